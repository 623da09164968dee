cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r02_recheck
timeout 900 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_ring.py -m gpu -q -p no:cacheprovider -k "not full_horizon and not full_ring" > gpurun_out/r02_recheck/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_recheck/pytest.log
tail -3 gpurun_out/r02_recheck/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3 | tee gpurun_out/r02_recheck/smoke.log
