#!/bin/bash
# ncu --set full of K6's two kernels on cfg3 (after the plain run exited 0).  Output under gpurun_out/$1.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_k6prof}
mkdir -p $O
timeout 300 python tools/profile_target.py cfg3 41 0 prof > $O/plain.log 2>&1 || { cat $O/plain.log; exit 1; }
cat $O/plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv python tools/profile_target.py cfg3 41 > $O/ncu_l.log 2>&1
for k in k_ring_cone k_ring_walls; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/full_$k python tools/profile_target.py cfg3 41 > $O/ncu_f_$k.log 2>&1
  python tools/ncu_lines.py $O/full_$k.ncu-rep 40 > $O/lines_$k.txt 2>&1
  ln -sf full_$k.ncu-rep $O/full_cfg3.ncu-rep
  python tools/ncu_summary.py $O cfg3 > $O/summary_$k.txt 2>&1
  ncu -i $O/full_$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>/dev/null
  rm -f $O/full_cfg3.ncu-rep $O/full_$k.ncu-rep
  cat $O/summary_$k.txt; head -25 $O/lines_$k.txt
done
