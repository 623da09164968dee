#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_5.log
timeout 300 ./tools/k1_variants > gpurun_out/k1_variants_2.log 2>&1
timeout 600 python bench.py --config cfg0 --steps 3 --warmup 3 > gpurun_out/bench_cfg0_b.json 2> gpurun_out/bench_cfg0_b.err
timeout 300 python tools/profile_target.py cfg3 21 > gpurun_out/plain_cfg3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 60 --log-file gpurun_out/launches_cfg3_r01.csv python tools/profile_target.py cfg3 21 > gpurun_out/ncu_cfg3_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_step_general -s 5 -c 1 -o gpurun_out/general_cfg3_r01 python tools/profile_target.py cfg3 21 > gpurun_out/ncu_cfg3_full.log 2>&1
timeout 300 python tools/profile_target.py cfg4 33 > gpurun_out/plain_cfg4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_analytic_tiled -c 1 -o gpurun_out/tiled_cfg4_r01 python tools/profile_target.py cfg4 33 > gpurun_out/ncu_cfg4_full.log 2>&1
ls -la gpurun_out | tail -30
