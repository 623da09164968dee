#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -p no:cacheprovider > gpurun_out/pytest_dv3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dv3.log
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 > gpurun_out/bench_dv_cfg4.json 2> gpurun_out/bench_dv_cfg4.err
