#!/bin/bash
# round 2 (c): full GPU suite after -fmad=false, the material parity path and K5;
# bench lines for cfg3 (K5 vs K4r), cfg5, cfg0
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_c
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ring.py tests/test_gpu_fastmath.py -m gpu -q -p no:cacheprovider -rA -x > $O/pytest_ring.log 2>&1; echo "rc=$?" >> $O/pytest_ring.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=15 > $O/pytest_all.log 2>&1; echo "rc=$?" >> $O/pytest_all.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --config cfg0 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg0.json 2> $O/bench_cfg0.err
