#!/bin/bash
# round 2: GPU test suite (+ smoke) on one box; logs under gpurun_out/$1
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_tests}
mkdir -p $O
nproc > $O/nproc.txt
timeout ${2:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=25 ${3:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
