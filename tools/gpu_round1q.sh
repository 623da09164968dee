#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "cfg2 or f32 or fp32 or fused or guard or golden" > gpurun_out/pytest_gpu_f32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_f32.log
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 3 > gpurun_out/bench_cfg2_b.json 2> gpurun_out/bench_cfg2_b.err
