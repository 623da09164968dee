#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for c in cfg5 cfg1 cfg3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${c}_e.json 2> gpurun_out/bench_${c}_e.err; done
