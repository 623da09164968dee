#!/bin/bash
# K4r role/IO timing: per-launch time vs steps per launch for the library and RING_SKIP variants
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/ringvar
mkdir -p $O
timeout 300 python tools/ring_step_probe.py > $O/probe_lib.log 2>&1
for v in ${RV:-8 16 24 56}; do
  timeout 300 python tools/ring_step_probe.py tools/_ringvar/libhygro_skip$v.so > $O/probe_skip$v.log 2>&1
done
