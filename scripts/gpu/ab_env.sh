#!/bin/bash
# A/B of an environment switch on the bench lines of the given configs:
# usage: ab_env.sh "<VAR=value>" "<configs>" [tag]   (B = the same run with the variable set)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${3:-ab}
for c in $2; do
  for arm in A B; do
    if [ $arm = B ]; then ENVV="$1"; else ENVV="DESPOT_AB_NONE=1"; fi
    env $ENVV timeout 300 python bench.py --config $c --no-cpu-baseline --no-all-cores-baseline > gpurun_out/ab_${TAG}_${arm}_c$c.json 2>/dev/null
    python - "$c" "$arm" "$TAG" <<'PY'
import json, sys
c, arm, tag = sys.argv[1:4]
try:
    d = json.loads(open(f"gpurun_out/ab_{tag}_{arm}_c{c}.json").read().strip().splitlines()[-1])
    ph = d["phases_ms"]
    print("c%s %s ms/step %.4f K1 %.4f K2 %.4f K3 %.4f e2e %.4g" % (c, arm, d["ms_per_step"], ph["K1_update"], ph["K2_expand_rollout"], ph["K3_finalize"], d["e2e"]["value"]))
except Exception as e:
    print("c%s %s parse failed %s" % (c, arm, e))
PY
  done
done
