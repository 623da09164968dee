#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_ring4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ring4.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3_i.json 2> gpurun_out/bench_cfg3_i.err
timeout 300 python tools/profile_target.py cfg3 41 > gpurun_out/plain_cfg3r.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring_tiled -s 2 -c 1 -o gpurun_out/ring_cfg3_r01d python tools/profile_target.py cfg3 41 > gpurun_out/ncu_cfg3_ring.log 2>&1
