#!/usr/bin/env python3
"""NEXT-2 of SURVEY §8(f): the paper's scalability studies as tree size per
planning time of the host tree driver on the GPU backend vs the same
driver on the CPU oracle backend (serial DESPOT analog), on synthetic beliefs
(`bench.py --plan --plan-study K|A`):

  * K sweep: navigation 13x13, K = 100 ... 5000, 1 s planning time.
  * |A| sweep: multi-agent RockSample (11,11), (15,15), (20,20),
    |A| = 256, 400, 625, fixed K.

One JSON line per (study, point, backend).  GPU box only.

  python scripts/next2_sweeps.py [--budget 1.0] [--K 100 500 1000 2000 5000] [--workers 1 8]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=1.0)
    ap.add_argument("--K", type=int, nargs="*", default=[100, 500, 1000, 2000, 5000])
    ap.add_argument("--A-K", type=int, default=500, help="the fixed K of the |A| sweep")
    ap.add_argument("--workers", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--studies", nargs="*", default=["K", "A"])
    args = ap.parse_args()
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--plan", "--plan-workers", *map(str, args.workers),
            "--plan-budget", str(args.budget)]
    rc = 0
    if "K" in args.studies:
        rc |= subprocess.call(base + ["--plan-study", "K", "--plan-K", *map(str, args.K)])
    if "A" in args.studies:
        rc |= subprocess.call(base + ["--plan-study", "A", "--K", str(args.A_K)])
    sys.exit(rc)


if __name__ == "__main__":
    main()
