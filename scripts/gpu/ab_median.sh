#!/bin/bash
# A/B of an environment switch by per-step medians (BENCH_STEP_LOG), arms
# alternated R times: usage ab_median.sh "<VAR=value>" <config> [steps] [R]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
C=$2; N=${3:-60}; R=${4:-2}
for r in $(seq 1 $R); do
  for arm in A B; do
    if [ $arm = B ]; then ENVV="$1"; else ENVV="DESPOT_AB_NONE=1"; fi
    env $ENVV BENCH_STEP_LOG=1 timeout 300 python bench.py --config $C --steps $N --warmup 5 --no-cpu-baseline --no-all-cores-baseline 2> gpurun_out/abm_err.txt > /dev/null
    python - "$arm" "$r" <<'PY'
import ast, statistics, sys
line = [l for l in open("gpurun_out/abm_err.txt") if l.startswith("step_ms")][-1]
v = ast.literal_eval(line[len("step_ms"):].strip())
v.sort()
print("%s r%s median %.4f p10 %.4f p90 %.4f" % (sys.argv[1], sys.argv[2], statistics.median(v), v[len(v)//10], v[9*len(v)//10]))
PY
  done
done
