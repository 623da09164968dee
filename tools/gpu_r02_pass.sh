#!/bin/bash
# round 2 full pass (cfg3 on K6, cfg4 on TMA tiles): GPU tests + smoke, bench lines for every config (with the CPU
# baselines), the reference arm (cfg1, cfg3), ncu launch lists and one --set full
# capture per config's dominant kernel (each ncu command only after its plain run
# exited 0).  Output under gpurun_out/$1.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_pass}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 1200 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg1.json 2> $O/bench_ref_cfg1.err
for c in cfg0 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 2 --ring-kernel 3 --no-cpu-baseline --no-e2e > $O/bench_cfg3_k5.json 2> $O/bench_cfg3_k5.err
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 2 --ring-kernel 1 --no-cpu-baseline --no-e2e > $O/bench_cfg3_k4r.json 2> $O/bench_cfg3_k4r.err
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 2 --tiled-load 1 --no-cpu-baseline --no-e2e > $O/bench_cfg4_cpasync.json 2> $O/bench_cfg4_cpasync.err
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --material-exact --no-cpu-baseline --no-e2e > $O/bench_cfg5_exact.json 2> $O/bench_cfg5_exact.err
timeout 900 python bench.py --impl reference --config cfg3 --steps 3 --warmup 1 > $O/bench_ref_cfg3.json 2> $O/bench_ref_cfg3.err
echo benches >> $O/status.txt
[ "${SKIP_PROF:-0}" = 1 ] && exit 0
lst() {   # cfg steps
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$1.csv python tools/profile_target.py $1 $2 > $O/ncu_l_$1.log 2>&1
}
full() {  # cfg steps kernel skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o $O/full_$1 python tools/profile_target.py $1 $2 > $O/ncu_f_$1.log 2>&1
  ncu -i $O/full_$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
  python tools/ncu_lines.py $O/full_$1.ncu-rep 30 > $O/lines_$1.txt 2>&1
  python tools/ncu_summary.py $O $1 > $O/summary_$1.txt 2>&1
  rm -f $O/full_$1.ncu-rep            # gpurun copies back <= 64 MiB
}
for c in "cfg1 4097" "cfg2 4097" "cfg0 4097" "cfg3 41" "cfg4 33" "cfg5 11"; do
  set -- $c
  timeout 600 python tools/profile_target.py $1 $2 > $O/plain_$1.log 2>&1 && lst $1 $2
done
echo lists >> $O/status.txt
full cfg1 4097 k_df_coupled 0
full cfg3 41 k_ring_walls 1
full cfg4 33 k_dv_tiled_tma 2
full cfg0 4097 k_dv_wall_halo 0
full cfg5 11 k_material_step 3
echo done >> $O/status.txt
