#!/bin/bash
# round-1 final pass (fourth session, after the restore): GPU tests, smoke, bench lines for all configs with the
# CPU baselines, the reference arm, launch lists, --set full captures of the changed kernels
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/final3
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in cfg0 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
echo benches >> $O/status.txt
lst() {   # cfg steps
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$1.csv python tools/profile_target.py $1 $2 > $O/ncu_l_$1.log 2>&1
}
full() {  # cfg steps kernel skip keep
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/full_$1 python tools/profile_target.py $1 $2 > $O/ncu_f_$1.log 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
  python tools/ncu_lines.py $O/full_$1.ncu-rep 40 > $O/lines_$1.txt 2>&1
  [ "$5" != keep ] && rm -f $O/full_$1.ncu-rep
}
lst cfg1 4097; lst cfg2 4097; lst cfg0 4097; lst cfg3 41; lst cfg4 33; lst cfg5 11
echo lists >> $O/status.txt
full cfg4 33 k_dv_tiled_stream 2 keep
full cfg0 4097 k_dv_wall_halo 0
full cfg3 41 k_ring_reg 1
full cfg5 11 k_material_step 3
echo done >> $O/status.txt
