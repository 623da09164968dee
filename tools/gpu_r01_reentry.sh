#!/bin/bash
# re-entry check: GPU tests, smoke, default bench, reference arm
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/reentry
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
