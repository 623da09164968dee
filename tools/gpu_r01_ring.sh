#!/bin/bash
# K4r experiment: ring tests, cfg3 bench line, per-launch timing vs steps per launch
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${RING_TAG:-ring}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_shard.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/ring_step_probe.py > $O/probe.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
