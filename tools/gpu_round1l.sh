#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_ring1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ring1.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_10.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3_g.json 2> gpurun_out/bench_cfg3_g.err
