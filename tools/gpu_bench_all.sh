#!/bin/bash
# One GPU call: bench.py lines for every BASELINE config + the reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 rc=$?" >> gpurun_out/bench_rc.log
for c in cfg0 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?" >> gpurun_out/bench_rc.log
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_cfg1.json 2> gpurun_out/bench_ref_cfg1.err; echo "ref rc=$?" >> gpurun_out/bench_rc.log
cat gpurun_out/bench_rc.log
