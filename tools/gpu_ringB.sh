#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for B in 7 5 4 3 2; do
  HYG_RING_B=$B timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_ringB$B.json 2> gpurun_out/bench_ringB$B.err
done
