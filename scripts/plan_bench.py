#!/usr/bin/env python3
"""Tree size per planning time (the paper's speedup metric) of the host
tree driver on the GPU backend vs the same driver on the CPU oracle backend
(serial DESPOT analog), SURVEY §8(f) NEXT-2.  Prints one JSON line per run.

  python scripts/plan_bench.py [--configs 1 2 3] [--budget 1.0] [--workers 1 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1802_06215_b200 import inputs  # noqa: E402
from paper_1802_06215_b200 import despot as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3])
    ap.add_argument("--budget", type=float, default=1.0)
    ap.add_argument("--workers", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    for cfg in args.configs:
        kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=args.K)
        rows = []
        gm = D.Model(kind, params)
        root = gm.belief_load(st, w, seed)
        for W in args.workers:
            c = D.search_config(workers=W, max_inflight=8 if W > 1 else 1, max_batch=64, batch_wait_us=300,
                                time_budget_s=args.budget, xi=0.95, c_a=0.3, c_o=0.1)
            r = gm.plan(root, c)
            r.update(backend="gpu", workers=W, config=cfg, K=len(w), nodes_per_s=r["nodes"] / r["seconds"],
                     leaves_per_batch=r["expanded"] / max(1, r["batches"]))
            rows.append(r)
            print(json.dumps(r), flush=True)
        if not args.no_oracle:
            import oracle
            from test_search_cpu import OracleBackend
            om = oracle.Model(kind, params)
            orr = om.belief_load(st, w, seed)
            u0, l0 = om.rollout_bounds(orr)
            be = OracleBackend(om)
            c = D.search_config(workers=1, max_inflight=1, max_batch=1, time_budget_s=args.budget, xi=0.95,
                                c_a=0.3, c_o=0.1)
            t = time.perf_counter()
            r, _ = D.search(be.problem(orr, u0, l0, K=len(w)), c)
            r.update(backend="oracle-serial", workers=1, config=cfg, K=len(w), nodes_per_s=r["nodes"] / r["seconds"],
                     wall=time.perf_counter() - t)
            print(json.dumps(r), flush=True)
            for g in rows:
                print(json.dumps({"config": cfg, "workers": g["workers"],
                                  "speedup_tree_size_per_time": g["nodes_per_s"] / r["nodes_per_s"]}), flush=True)
        gm.close()


if __name__ == "__main__":
    main()
