#!/bin/bash
# ncu launch lists + --set full captures of the current kernels (each ncu run after its plain run exited 0)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/prof3
mkdir -p $O
prof() {   # cfg steps kernel_regex skip
  local c=$1 st=$2 k=$3 sk=$4
  timeout 600 python tools/profile_target.py $c $st > $O/plain_$c.log 2>&1 || { echo "plain $c failed" >> $O/status.txt; return; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$c.csv python tools/profile_target.py $c $st > $O/ncu_l_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o $O/full_$c python tools/profile_target.py $c $st > $O/ncu_f_$c.log 2>&1
  ncu -i $O/full_$c.ncu-rep --page raw --csv > $O/raw_$c.csv 2>/dev/null
  python tools/ncu_lines.py $O/full_$c.ncu-rep 40 > $O/lines_$c.txt 2>&1
  [ "$c" != "${KEEP:-cfg4}" ] && rm -f $O/full_$c.ncu-rep
  echo "$c done" >> $O/status.txt
}
prof ${1:-cfg4} ${2:-33} ${3:-k_dv_tiled_stream} ${4:-2}
[ -n "$5" ] && prof cfg3 41 k_ring_reg 1
[ -n "$5" ] && prof cfg5 11 k_material_step 3
[ -n "$5" ] && prof cfg0 4097 k_dv_wall_split 0
echo all >> $O/status.txt
