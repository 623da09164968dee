#!/bin/bash
# overlapped halo refresh check: shard tests (loopback device payloads, two processes on one GPU), long-wall tests, cfg4 bench
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${1:-r02_overlap}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -rA -k "shard or long or tiled or cfg4 or payload or ranks or dv" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
grep -E "FAILED|ERROR|passed|failed|rc=" $O/pytest.log | tail -8
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python -c "
import json
d = json.loads(open('$O/bench_cfg4.json').read().strip().splitlines()[-1]); print('cfg4 value %.4g' % d['value'])"
