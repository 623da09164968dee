#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 120 ./tools/latency_probe > gpurun_out/latency_probe.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_6.log
for c in cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${c}_b.json 2> gpurun_out/bench_${c}_b.err; done
timeout 300 python tools/profile_target.py cfg4 33 > gpurun_out/plain_cfg4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_analytic_tiled -c 1 -o gpurun_out/tiled_cfg4_r01b python tools/profile_target.py cfg4 33 > gpurun_out/ncu_cfg4_full_b.log 2>&1
ls gpurun_out | tail -5
