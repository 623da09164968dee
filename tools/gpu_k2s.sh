#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_material.py -q -p no:cacheprovider -k "dv_wall or cfg0 or nonlinear or analytic" > gpurun_out/pytest_k2s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k2s.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_k2s.log 2>&1
timeout 600 python bench.py --config cfg0 --steps 3 --warmup 3 > gpurun_out/bench_k2s_cfg0.json 2> gpurun_out/bench_k2s_cfg0.err
