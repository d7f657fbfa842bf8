#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
# (logs under gpurun_out/sanitize/, copied to profiles/r02/ when read back)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/sanitize; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in fused k1_dense rank sparse merge; do
    extra=""
    timeout 600 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_cases.py $c > $OUT/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a $OUT/summary.txt
  done
done
