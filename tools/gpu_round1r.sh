#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "cfg0 or cfg4 or tiled or fastmath or nonlinear or analytic or golden" > gpurun_out/pytest_gpu_k2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_k2.log
for c in cfg0 cfg4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${c}_j.json 2> gpurun_out/bench_${c}_j.err; done
