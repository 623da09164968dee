#!/bin/bash
# shard device-payload tests + source-level ncu captures of K4r and K3w
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/t1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shard.py -q -p no:cacheprovider > $O/pytest_shard.log 2>&1; echo "rc=$?" >> $O/pytest_shard.log
timeout 300 python tools/profile_target.py cfg3 41 > $O/plain_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring_reg -s 1 -c 1 -o $O/full_cfg3 python tools/profile_target.py cfg3 41 > $O/ncu_cfg3.log 2>&1
timeout 300 python tools/profile_target.py cfg4 33 > $O/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dv_tiled_stream -s 2 -c 1 -o $O/full_cfg4 python tools/profile_target.py cfg4 33 > $O/ncu_cfg4.log 2>&1
echo done >> $O/status.txt
