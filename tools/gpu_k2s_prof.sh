#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
timeout 300 python tools/profile_target.py cfg0 4097 > gpurun_out/prof/plain_cfg0.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dv_wall_split -s 0 -c 1 -o gpurun_out/prof/k2s_cfg0 python tools/profile_target.py cfg0 4097 > gpurun_out/prof/ncu_k2s.log 2>&1
