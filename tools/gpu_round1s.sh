#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_material.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_edges.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_edges.log
