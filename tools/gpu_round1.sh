cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_3.log
timeout 300 ./tools/k1_variants > gpurun_out/k1_variants.log 2>&1; echo "rc=$?" >> gpurun_out/k1_variants.log
timeout 300 python tools/profile_target.py cfg1 > gpurun_out/plain_cfg1.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_r01.csv python tools/profile_target.py cfg1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_df_coupled -c 1 -o gpurun_out/k1_full_r01 python tools/profile_target.py cfg1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
ls -la gpurun_out
