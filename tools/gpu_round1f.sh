#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_8.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3_d.json 2> gpurun_out/bench_cfg3_d.err
timeout 300 python tools/profile_target.py cfg3 21 > gpurun_out/plain_cfg3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_building_step -s 5 -c 1 -o gpurun_out/building_cfg3_r01d python tools/profile_target.py cfg3 21 > gpurun_out/ncu_cfg3_d.log 2>&1
