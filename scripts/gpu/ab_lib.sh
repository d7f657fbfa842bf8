#!/bin/bash
# A/B of two builds of the library by per-step medians (BENCH_STEP_LOG):
# usage: ab_lib.sh <libA.so> <libB.so> <config> [steps] [R]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
A=$1; B=$2; C=$3; N=${4:-30}; R=${5:-2}
for r in $(seq 1 $R); do
  for arm in A B; do
    L=$A; [ $arm = B ] && L=$B
    DESPOT_LIB=$L BENCH_STEP_LOG=1 timeout 300 python bench.py --config $C --steps $N --warmup 5 --no-cpu-baseline --no-all-cores-baseline 2> gpurun_out/abl_err.txt > gpurun_out/abl_$arm.json
    python - "$arm" "$r" <<'PY'
import ast, json, statistics, sys
line = [l for l in open("gpurun_out/abl_err.txt") if l.startswith("step_ms")][-1]
v = sorted(ast.literal_eval(line[len("step_ms"):].strip()))
d = json.loads(open("gpurun_out/abl_%s.json" % sys.argv[1]).read().strip().splitlines()[-1])
print("%s r%s median %.4f p10 %.4f p90 %.4f K2 %.4f" % (sys.argv[1], sys.argv[2], statistics.median(v), v[len(v)//10], v[9*len(v)//10], d["phases_ms"]["K2_expand_rollout"]))
PY
  done
done
