#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_4.log
bash tools/gpu_bench_all.sh
