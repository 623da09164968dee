#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_material.py -q -p no:cacheprovider -s > gpurun_out/pytest_gpu_mat2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_mat2.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5_a.json 2> gpurun_out/bench_cfg5_a.err
timeout 300 python tools/profile_target.py cfg5 5 > gpurun_out/plain_cfg5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_star_tables -s 3 -c 1 -o gpurun_out/star_cfg5_r01 python tools/profile_target.py cfg5 5 > gpurun_out/ncu_cfg5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg5.csv python tools/profile_target.py cfg5 5 > gpurun_out/ncu_cfg5_l.log 2>&1
