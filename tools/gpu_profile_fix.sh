#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
for spec in "cfg1 4097 k_df_coupled" "cfg2 4097 k_df_coupled" "cfg0 4097 k_df_analytic_walls"; do
  set -- $spec
  timeout 600 python tools/profile_target.py $1 $2 > gpurun_out/prof/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -c 1 -o gpurun_out/prof/full_$1 python tools/profile_target.py $1 $2 > gpurun_out/prof/ncu_f_$1.log 2>&1
done
