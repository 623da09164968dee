#!/bin/bash
# round 2: compute-sanitizer passes over the smallest case of every kernel family
# (tools/sanitize_target.py), one tool per case list; summaries under gpurun_out/r02_san
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r02_san
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${1:-racecheck synccheck}; do
  for c in k1 k2h k3w k5 k4r material; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_target.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" >> $O/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" $O/${tool}_$c.log | tail -3 >> $O/summary.txt
  done
done
