#!/bin/bash
# ncu source-level (CUDA line) instruction and stall attribution of K2 for a config
cd "${GRAFT_REPO_ROOT:-/root/repo}"
C=$1; TAG=$2; shift 2
O=gpurun_out/ncu; mkdir -p $O
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/$TAG python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-all-cores-baseline "$@" > $O/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source cuda > $O/${TAG}_cuda.csv 2>/dev/null
rm -f $O/$TAG.ncu-rep
