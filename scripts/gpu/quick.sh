#!/bin/bash
# quick GPU check: parity tests selected by -k, then bench lines of the given configs
# usage: quick.sh "<pytest -k expr>" "<configs>" [tag]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${3:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_$TAG.txt 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_$TAG.txt
for c in $2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-all-cores-baseline > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err
  echo "bench c$c rc=$?"
  python - "$c" "$TAG" <<'PY'
import json, sys
c, tag = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bench_{tag}_c{c}.json").read().strip().splitlines()[-1])
    print("c%s value %.4g ms/step %.4f K2 %.4f frac %.3f e2e %.4g" % (c, d["value"], d["ms_per_step"], d["phases_ms"]["K2_expand_rollout"], d["roofline"]["frac"], d["e2e"]["value"]))
except Exception as e:
    print("c%s parse failed %s" % (c, e))
PY
done
