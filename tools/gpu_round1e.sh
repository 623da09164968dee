#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_7.log
for c in cfg0 cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${c}_c.json 2> gpurun_out/bench_${c}_c.err; done
timeout 300 python tools/profile_target.py cfg3 21 > gpurun_out/plain_cfg3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_building_step -s 5 -c 1 -o gpurun_out/building_cfg3_r01 python tools/profile_target.py cfg3 21 > gpurun_out/ncu_cfg3_b.log 2>&1
timeout 300 python tools/profile_target.py cfg0 4097 > gpurun_out/plain_cfg0.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_analytic_walls -c 1 -o gpurun_out/walls_cfg0_r01 python tools/profile_target.py cfg0 4097 > gpurun_out/ncu_cfg0.log 2>&1
timeout 300 python tools/profile_target.py cfg4 33 > gpurun_out/plain_cfg4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_analytic_tiled -c 1 -o gpurun_out/tiled_cfg4_r01c python tools/profile_target.py cfg4 33 > gpurun_out/ncu_cfg4_c.log 2>&1
ls gpurun_out | tail -3
