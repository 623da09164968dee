#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_material.py tests/test_gpu_scenarios.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_mat4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_mat4.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5_g.json 2> gpurun_out/bench_cfg5_g.err
