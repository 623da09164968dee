#!/bin/bash
# d(v) instruction trim: full GPU suite, cfg0/cfg4 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/${DV_TAG:-dv4}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in cfg4 cfg0; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
