#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
RING_TAG=${RING_TAG:-ring4} bash tools/gpu_r01_ring.sh
timeout 300 python tools/ring_prof_probe.py tools/_ringvar/libhygro_skip0p.so > gpurun_out/${RING_TAG:-ring4}/ringprof.log 2>&1
