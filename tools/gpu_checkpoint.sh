#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_ckpt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ckpt.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_ckpt.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ckpt.log
timeout 900 python bench.py > gpurun_out/bench_default_ckpt.json 2> gpurun_out/bench_default_ckpt.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_ckpt.json 2> gpurun_out/bench_ref_ckpt.err
