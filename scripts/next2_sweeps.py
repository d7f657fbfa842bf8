#!/usr/bin/env python3
"""NEXT-2 of SURVEY §8(f): the paper's scalability studies as tree size per
planning time (its speedup metric) of the host tree driver on the GPU
backend vs the same driver on the CPU oracle backend (serial DESPOT analog),
on synthetic beliefs:

  * K sweep: navigation 13x13, K = 100 ... 5000, 1 s planning
    time: nodes/s, search depth, speedup.
  * |A| sweep: multi-agent RockSample (11,11), (15,15), (20,20),
    |A| = 256, 400, 625, fixed K.

One JSON line per (study, point, backend).  GPU box only.

  python scripts/next2_sweeps.py [--budget 1.0] [--K 100 500 1000 2000 5000] [--workers 8]
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


def run_point(study, point, kind, params, st, w, seed, budget, workers, oracle_budget):
    rows = []
    gm = D.Model(kind, params)
    root = gm.belief_load(st, w, seed)
    for W in workers:
        c = D.search_config(workers=W, max_inflight=8 if W > 1 else 1, max_batch=64, batch_wait_us=300,
                            time_budget_s=budget, xi=0.95, c_a=0.3, c_o=0.1)
        r = gm.plan(root, c)
        r.update(study=study, point=point, backend="gpu", workers=W, K=len(w), A=gm.A,
                 nodes_per_s=r["nodes"] / r["seconds"])
        rows.append(r)
        print(json.dumps(r), flush=True)
    gm.close()
    import oracle
    from test_search_cpu import OracleBackend
    om = oracle.Model(kind, params)
    orr = om.belief_load(st, w, seed)
    u0, l0 = om.rollout_bounds(orr)
    be = OracleBackend(om)
    c = D.search_config(workers=1, max_inflight=1, max_batch=1, time_budget_s=oracle_budget, xi=0.95, c_a=0.3,
                        c_o=0.1)
    t = time.perf_counter()
    r, _ = D.search(be.problem(orr, u0, l0, K=len(w)), c)
    r.update(study=study, point=point, backend="oracle-serial", workers=1, K=len(w), A=om.A,
             nodes_per_s=r["nodes"] / r["seconds"], wall=time.perf_counter() - t)
    print(json.dumps(r), flush=True)
    for g in rows:
        print(json.dumps({"study": study, "point": point, "workers": g["workers"],
                          "speedup_tree_size_per_time": g["nodes_per_s"] / r["nodes_per_s"],
                          "gpu_max_depth": g["max_depth"], "oracle_max_depth": r["max_depth"]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=1.0)
    ap.add_argument("--oracle-budget", type=float, default=None, help="default: --budget")
    ap.add_argument("--K", type=int, nargs="*", default=[100, 500, 1000, 2000, 5000])
    ap.add_argument("--A-K", type=int, default=500, help="the fixed K of the |A| sweep")
    ap.add_argument("--workers", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--studies", nargs="*", default=["K", "A"])
    args = ap.parse_args()
    ob = args.oracle_budget or args.budget
    if "K" in args.studies:
        for K in args.K:
            kind, params, st, w, seed, _ = inputs.config_inputs(3, K=K)
            run_point("K_nav13", K, kind, params, st, w, seed, args.budget, args.workers, ob)
    if "A" in args.studies:
        for n, m in ((11, 11), (15, 15), (20, 20)):  # |A| = (5 + m)^2 = 256, 400, 625
            params = inputs.rocksample_params(n, m, 2, D=20)
            st = inputs.rocksample_belief(n, m, 2, args.A_K, 1002)
            w = inputs.weights(args.A_K, 1002)
            run_point("A_mars", f"MARS({n},{n}) |A|={(5 + m) ** 2}", "rocksample", params, st, w, 1002, args.budget,
                      args.workers, ob)


if __name__ == "__main__":
    main()
