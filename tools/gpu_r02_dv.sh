#!/bin/bash
# d(v) arithmetic change check: fastmath / parity / golden / determinism / shard / edge tests, then cfg4 and cfg0 bench lines.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_dv}
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_determinism.py tests/test_gpu_shard.py tests/test_gpu_edges.py tests/test_gpu_adapter.py -m gpu -q -p no:cacheprovider -rA > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
grep -E "FAILED|ERROR|passed|failed|rc=" $O/pytest.log | tail -15
for c in cfg4 cfg0; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  python - <<PY
import json
try:
    d = json.loads(open("$O/bench_$c.json").read().strip().splitlines()[-1])
    print("$c value %.4g  %s rate %.4g frac %.3f clocks %s" % (d["value"], d["roofline"]["kernel"], d["roofline"]["kernel_node_updates_per_s"], d["roofline"]["frac"], d["clocks"]))
except Exception as e:
    print("$c failed", e); print(open("$O/bench_$c.err").read()[-2000:])
PY
done
