#!/bin/bash
# K2h (halo variant of the single-wall d(v) march, configs[0]): GPU tests, bench line, launch list, ncu capture
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/k2h
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config cfg0 --steps 10 --warmup 3 > $O/bench_cfg0.json 2> $O/bench_cfg0.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_cfg0.csv python tools/profile_target.py cfg0 4097 > $O/ncu_l_cfg0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dv_wall_halo -c 1 -o $O/full_cfg0 python tools/profile_target.py cfg0 4097 > $O/ncu_f_cfg0.log 2>&1
ncu -i $O/full_cfg0.ncu-rep --page raw --csv > $O/raw_cfg0.csv 2>/dev/null
python tools/ncu_lines.py $O/full_cfg0.ncu-rep 30 > $O/lines_cfg0.txt 2>&1
rm -f $O/full_cfg0.ncu-rep
for r in 1 2; do timeout 120 python tools/dv_time_probe.py; timeout 120 python tools/dv_time_probe.py tools/_ringvar/libhygro_SQRT.so; done > $O/probe.txt 2>&1
