#!/bin/bash
# source-level ncu captures: K1 (cfg1), K2s (cfg0), K4r (cfg3) after the round-1 changes
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/prof2
mkdir -p $O
prof() {   # cfg steps kernel_regex skip
  local c=$1 st=$2 k=$3 sk=$4
  timeout 600 python tools/profile_target.py $c $st > $O/plain_$c.log 2>&1 || { echo "plain $c failed" >> $O/status.txt; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o $O/full_$c python tools/profile_target.py $c $st > $O/ncu_f_$c.log 2>&1
  echo "$c done" >> $O/status.txt
}
prof cfg1 4097 k_df_coupled 0
prof cfg0 4097 k_dv_wall_split 0
prof cfg3 41 k_ring_reg 1
