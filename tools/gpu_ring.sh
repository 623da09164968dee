#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "ring or cfg3" > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ring.log
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_ring_cfg3.json 2> gpurun_out/bench_ring_cfg3.err
