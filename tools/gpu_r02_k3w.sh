#!/bin/bash
# K3w TMA tiles check: the long-wall tests, then cfg4 bench A/B (TMA tiles vs cp.async).  Output under gpurun_out/$1.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_k3w}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider -rA -k "long or tiled or dv or cfg4" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
for k in 0 1; do
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --tiled-load $k --no-cpu-baseline --no-e2e > $O/bench_cfg4_l$k.json 2> $O/bench_cfg4_l$k.err
  python - <<PY
import json
try:
    d = json.loads(open("$O/bench_cfg4_l$k.json").read().strip().splitlines()[-1])
    print("tiled_load $k value %.4g  %s rate %.4g frac %.3f clocks %s" % (d["value"], d["roofline"]["kernel"], d["roofline"]["kernel_node_updates_per_s"], d["roofline"]["frac"], d["clocks"]))
except Exception as e:
    print("tiled_load $k failed", e); print(open("$O/bench_cfg4_l$k.err").read()[-2000:])
PY
done
