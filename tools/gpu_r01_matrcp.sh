#!/bin/bash
# material step with reciprocal quotients: GPU tests, cfg5 bench line, launch list
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/matrcp
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg5.csv python tools/profile_target.py cfg5 11 > $O/ncu_l_cfg5.log 2>&1
