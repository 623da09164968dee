#!/bin/bash
# one --set full capture of the K3w interior kernel (after a clean run)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
timeout 300 python tools/profile_target.py cfg4 33 > gpurun_out/prof/plain_cfg4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dv_tiled -s 2 -c 1 -o gpurun_out/prof/dv3_cfg4 python tools/profile_target.py cfg4 33 > gpurun_out/prof/ncu_dv3_cfg4.log 2>&1
