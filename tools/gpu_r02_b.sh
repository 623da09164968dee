#!/bin/bash
# round 2 (b): new parity-depth + fixture/acceptance tests, the bench line with
# the new cpu_baseline, and the reference arm
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_b
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rA --durations=20 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref_cfg1.json 2> $O/bench_ref_cfg1.err
timeout 900 python bench.py --impl reference --config cfg3 --steps 3 --warmup 1 > $O/bench_ref_cfg3.json 2> $O/bench_ref_cfg3.err
