#!/bin/bash
# K2s/K2w/K3w (warp-register d(v) kernels): parity tests, then cfg0/cfg4 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_edges.py tests/test_gpu_shard.py tests/test_gpu_material.py -q -p no:cacheprovider > gpurun_out/pytest_dv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dv.log
timeout 600 python bench.py --config cfg0 --steps 3 --warmup 3 > gpurun_out/bench_dv_cfg0.json 2> gpurun_out/bench_dv_cfg0.err
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/bench_dv_cfg4.json 2> gpurun_out/bench_dv_cfg4.err
