#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dv_wall or cfg0" > gpurun_out/pytest_dv2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dv2.log
timeout 300 python tools/profile_target.py cfg0 4097 > gpurun_out/prof/plain_cfg0.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dv_wall -s 0 -c 1 -o gpurun_out/prof/dv2_cfg0 python tools/profile_target.py cfg0 4097 > gpurun_out/prof/ncu_dv2_cfg0.log 2>&1
