#!/bin/bash
# round-1 final pass: GPU tests, smoke, bench lines for all configs, launch lists and
# one --set full capture per changed kernel (each ncu run after its plain run exited 0)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in cfg0 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
prof() {   # cfg steps kernel_regex skip
  local c=$1 st=$2 k=$3 sk=$4
  timeout 600 python tools/profile_target.py $c $st > $O/plain_$c.log 2>&1 || { echo "plain $c failed" >> $O/status.txt; return; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$c.csv python tools/profile_target.py $c $st > $O/ncu_l_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o $O/full_$c python tools/profile_target.py $c $st > $O/ncu_f_$c.log 2>&1
  echo "$c done" >> $O/status.txt
}
prof cfg0 4097 k_dv_wall_split 0
prof cfg3 41 k_ring_reg 1
prof cfg4 33 k_dv_tiled_stream 2
