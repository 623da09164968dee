#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scenarios.py tests/test_gpu_adapter.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_scen1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_scen1.log
