#!/bin/bash
# one `ncu --set full` capture of K2 for the given config (raw + source pages)
# usage: ncu_k2.sh <config> <tag> [extra bench args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
C=$1; TAG=$2; shift 2
O=gpurun_out/ncu; mkdir -p $O
timeout 900 python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-all-cores-baseline "$@" > $O/plain_${TAG}.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_${TAG} python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-all-cores-baseline "$@" > $O/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i $O/k2_${TAG}.ncu-rep --page raw --csv > $O/k2_${TAG}_raw.csv 2>/dev/null
ncu -i $O/k2_${TAG}.ncu-rep --page source --csv --print-source sass > $O/k2_${TAG}_sass.csv 2>/dev/null
ncu -i $O/k2_${TAG}.ncu-rep --page details --csv > $O/k2_${TAG}_details.csv 2>/dev/null
ls -la $O
