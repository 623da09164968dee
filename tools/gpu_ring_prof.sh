#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
timeout 300 python tools/profile_target.py cfg3 41 > gpurun_out/prof/plain_cfg3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ring_reg -s 1 -c 1 -o gpurun_out/prof/ringreg_cfg3 python tools/profile_target.py cfg3 41 > gpurun_out/prof/ncu_ringreg.log 2>&1
