#!/bin/bash
# round 2 (f): K5 with producer warp + zone partial sums: ring tests, cfg3 timing, ncu lines
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_f
mkdir -p $O
timeout 420 python -m pytest tests/test_gpu_ring.py tests/test_gpu_shard.py -m gpu -q -p no:cacheprovider -rA -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 180 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/k5.json 2> $O/k5.err
HYG_DEBUG_RING_SKIP=1 timeout 180 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/k5_nohalo.json 2> $O/k5_nohalo.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ring_pipe -s 2 -c 1 -o $O/k5 python tools/profile_target.py cfg3 61 > $O/ncu.log 2>&1
ncu -i $O/k5.ncu-rep --page raw --csv > $O/k5_raw.csv 2>/dev/null
python tools/ncu_lines.py $O/k5.ncu-rep 45 > $O/k5_lines.txt 2>&1
