#!/bin/bash
# one `ncu --set full` capture of the first matching kernel of a bench config
# usage: ncu_kernel.sh <config> <kernel regex> <tag> [extra bench args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
C=$1; K=$2; TAG=$3; shift 3
O=gpurun_out/ncu; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $O/$TAG python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline --no-all-cores-baseline "$@" > $O/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i $O/$TAG.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ncu -i $O/$TAG.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>/dev/null
rm -f $O/$TAG.ncu-rep
