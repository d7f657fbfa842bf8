#!/usr/bin/env python3
"""Per-unit instruction figure of the dominant kernel (K2) per BASELINE config:
thread-instructions per scenario-step = ncu smsp__thread_inst_executed.sum of
one K2 launch / the scenario-steps of that batch.  Runs, per config, one
bench.py pass without ncu (for the step count), then the same command under
`ncu --metrics` (one GPU), and writes profiles/r01/i_step.json, which
bench.py reads for its ALU roofline.  GPU box only.

  python scripts/measure_istep.py [--configs 1 2 3 4 5]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench_cmd(cfg):
    c = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "1", "--warmup", "3",
         "--no-cpu-baseline"]
    if cfg == 5:
        c += ["--K", "4096"]
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "i_step.json"))
    args = ap.parse_args()
    res = {}
    if os.path.exists(args.out):
        res = json.load(open(args.out))
    for cfg in args.configs:
        out = subprocess.run(bench_cmd(cfg), capture_output=True, text=True, timeout=600)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if out.returncode or not line:
            print(json.dumps({"config": cfg, "error": out.stderr[-400:]}), flush=True)
            continue
        d = json.loads(line[0])
        steps = d["config"]["scenario_steps_per_batch"]
        kern = d["roofline"]["kernel"]
        csvp = f"/tmp/istep_{cfg}.csv"
        ncu = ["ncu", "--metrics", "smsp__thread_inst_executed.sum,smsp__inst_executed.sum,gpu__time_duration.sum",
               "--clock-control", "none", "-k", f"regex:{kern}", "--csv", "--log-file", csvp] + bench_cmd(cfg)
        r = subprocess.run(ncu, capture_output=True, text=True, timeout=1200)
        if r.returncode:
            print(json.dumps({"config": cfg, "error": r.stderr[-400:]}), flush=True)
            continue
        text = open(csvp).read()
        text = text[text.index('"ID"'):]  # skip ncu's own log lines before the CSV header
        rows = list(csv.DictReader(io.StringIO(text)))
        vals, units = {}, {}
        for row in rows:
            vals.setdefault(row["ID"], {})[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
            units[row["Metric Name"]] = row.get("Metric Unit", "")
        # the timed step's launch is the last one (warm-ups first); every launch has the same work
        last = vals[max(vals, key=int)]
        ti = last["smsp__thread_inst_executed.sum"]
        res[str(cfg)] = {"kernel": kern, "thread_inst_per_launch": ti, "scenario_steps_per_batch": steps,
                         "i_step": ti / steps, "warp_inst_per_launch": last["smsp__inst_executed.sum"],
                         "ncu_duration": last["gpu__time_duration.sum"], "ncu_duration_unit": units["gpu__time_duration.sum"],
                         "workload": d["config"]["workload"]}
        print(json.dumps({"config": cfg, **res[str(cfg)]}), flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
