#!/bin/bash
# K6 (k_ring_split.cuh) check: ring parity / determinism / shard tests, then cfg3 bench A/B
# (K6 default vs K4r) with per-kernel stats.  Output under gpurun_out/$1.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_k6}
mkdir -p $O
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests/test_gpu_ring.py tests/test_gpu_determinism.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider -rA -k "${TESTK:-not full_horizon}" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
  tail -5 $O/pytest.log
fi
for k in ${KERNELS:-0 1}; do
  timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --ring-kernel $k --no-cpu-baseline --no-e2e > $O/bench_cfg3_k$k.json 2> $O/bench_cfg3_k$k.err
  python - <<PY
import json
try:
    d = json.loads(open("$O/bench_cfg3_k$k.json").read().strip().splitlines()[-1])
    print("kernel $k value %.4g  %s rate %.4g share %.3f frac %.3f" % (d["value"], d["roofline"]["kernel"], d["roofline"]["kernel_node_updates_per_s"], d["roofline"]["kernel_share_of_step"], d["roofline"]["frac"]))
except Exception as e:
    print("kernel $k failed", e); print(open("$O/bench_cfg3_k$k.err").read()[-2000:])
PY
done
for d in ${DEPTHS:-1 2 3}; do
  timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --ring-depth $d --no-cpu-baseline --no-e2e > $O/bench_cfg3_d$d.json 2> $O/bench_cfg3_d$d.err
  python - <<PY
import json
try:
    d = json.loads(open("$O/bench_cfg3_d$d.json").read().strip().splitlines()[-1])
    print("depth $d value %.4g  %s rate %.4g share %.3f" % (d["value"], d["roofline"]["kernel"], d["roofline"]["kernel_node_updates_per_s"], d["roofline"]["kernel_share_of_step"]))
except Exception as e:
    print("depth $d failed", e); print(open("$O/bench_cfg3_d$d.err").read()[-2000:])
PY
done
for k in ${KERNELS:-0 1}; do
  timeout 300 python tools/profile_target.py cfg3 801 $k prof > $O/stats_k$k.txt 2>&1; cat $O/stats_k$k.txt
done
