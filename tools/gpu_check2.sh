#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/check2
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 300 python tools/profile_target.py cfg3 41 > $O/plain_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring_reg -s 1 -c 1 -o $O/full_cfg3 python tools/profile_target.py cfg3 41 > $O/ncu_f_cfg3.log 2>&1
