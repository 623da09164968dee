#!/bin/bash
# round 2 (g): K5 tests, phase stamps, cfg3 timing K5 vs K4r
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_g
mkdir -p $O
timeout 420 python -m pytest tests/test_gpu_ring.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 200 python tools/ring_pipe_prof.py tools/_ringvar/libhygro_prof.so > $O/prof.txt 2>&1
timeout 180 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/k5.json 2> $O/k5.err
