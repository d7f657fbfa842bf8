#!/usr/bin/env python3
"""NEXT-3 of SURVEY §8(f): the driving config with 6 / 12 / 20 pedestrians
 and the two kernel variants -- factored warp per
scenario (lanes = pedestrians + car) vs thread per scenario -- at
the full batch (64 roots x K=500) and a small one (8 roots x K=64, where the
factored kernel's extra parallelism matters), plus the grouped kernel (a lane
group per scenario, several scenarios per warp).  One JSON line per run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for K in (500, 64):
    for peds in (6, 12, 20):
        for variant in ("warp", "group", "pair", "thread"):
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "4", "--peds", str(peds), "--K", str(K),
                   "--car-variant", variant, "--steps", "10", "--warmup", "3", "--no-cpu-baseline"]
            out = subprocess.run(cmd, capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(json.dumps({"peds": peds, "K": K, "variant": variant, "error": out.stderr[-400:]}), flush=True)
                continue
            d = json.loads(line[0])
            print(json.dumps({"peds": peds, "K": K, "variant": variant, "value": d["value"],
                              "ms_per_step": d["ms_per_step"], "k2_ms": d["phases_ms"]["K2_expand_rollout"]}),
                  flush=True)
