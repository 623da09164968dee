#!/bin/bash
# round-1 profiling pass: per config a launch list and one --set full capture of
# its dominant kernel (each ncu command only after the same command exited 0)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
run() {   # cfg steps kernel_regex
  local c=$1 st=$2 k=$3
  timeout 600 python tools/profile_target.py $c $st > gpurun_out/prof/plain_$c.log 2>&1 || { echo "plain $c failed" >> gpurun_out/prof/status.txt; return; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/prof/launches_$c.csv python tools/profile_target.py $c $st > gpurun_out/prof/ncu_l_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof/full_$c python tools/profile_target.py $c $st > gpurun_out/prof/ncu_f_$c.log 2>&1
  echo "$c done" >> gpurun_out/prof/status.txt
}
run cfg1 4097 k_df_coupled
run cfg2 4097 k_df_coupled
run cfg0 4097 k_df_analytic_walls
run cfg3 41 k_ring_tiled
run cfg4 33 k_df_analytic_tiled
run cfg5 5 k_material_step
