cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_stubprof; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ring_stub -s 1 -c 1 -o $O/full_stub python tools/profile_target.py cfg3 81 > $O/ncu.log 2>&1
python tools/ncu_lines.py $O/full_stub.ncu-rep 30 > $O/lines.txt 2>&1
ln -sf full_stub.ncu-rep $O/full_cfg3.ncu-rep; echo > $O/launches_cfg3.csv
python tools/ncu_summary.py $O cfg3 > $O/summary.txt 2>&1
rm -f $O/full_cfg3.ncu-rep $O/full_stub.ncu-rep
cat $O/summary.txt | head -16; head -30 $O/lines.txt
