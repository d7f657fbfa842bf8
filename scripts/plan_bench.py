#!/usr/bin/env python3
"""Tree size per planning time (the paper's speedup metric) of the host
tree driver on the GPU backend vs the same driver on the CPU oracle backend
(serial DESPOT analog): `bench.py --plan` for the
BASELINE configs.  Prints one JSON line per run.

  python scripts/plan_bench.py [--configs 1 2 3 4] [--budget 1.0] [--workers 1 4 8]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3])
    ap.add_argument("--budget", type=float, default=1.0)
    ap.add_argument("--workers", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--plan", "--plan-study", "configs",
           "--plan-configs", *map(str, args.configs), "--plan-workers", *map(str, args.workers),
           "--plan-budget", str(args.budget)]
    if args.K:
        cmd += ["--K", str(args.K)]
    if args.no_oracle:
        cmd += ["--no-cpu-baseline"]
    sys.exit(subprocess.call(cmd))


if __name__ == "__main__":
    main()
