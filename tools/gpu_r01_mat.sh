#!/bin/bash
# material functor on fast exp/log/div: material + fastmath + scenario GPU tests, cfg5 bench line
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/mat
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_material.py tests/test_gpu_scenarios.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
