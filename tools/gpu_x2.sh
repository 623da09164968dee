#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_golden.py -q -p no:cacheprovider > gpurun_out/pytest_x2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x2.log
timeout 600 python bench.py --config cfg2 --steps 3 --warmup 3 > gpurun_out/bench_x2_cfg2.json 2> gpurun_out/bench_x2_cfg2.err
