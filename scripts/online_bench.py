#!/usr/bin/env python3
"""NEXT-4 of SURVEY §8(f): closed-loop episodes (plan -> act in the world ->
particle-filter update, paper_1802_06215_b200/online.py) on the GPU planner,
at several planning-time budgets: mean discounted return, steps, planning time
per step, tree size.  One JSON line per (model, budget).  GPU box only.

  python scripts/online_bench.py [--episodes 8] [--budgets 0.02 0.1 0.5] [--steps 40]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1802_06215_b200 import inputs, online  # noqa: E402
from paper_1802_06215_b200.despot import Model, search_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--episodes", type=int, default=8)
    ap.add_argument("--budgets", type=float, nargs="*", default=[0.02, 0.1, 0.5])
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--K", type=int, default=500)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--models", nargs="*", default=["rs78", "nav13"])
    args = ap.parse_args()
    for name in args.models:
        if name == "rs78":
            n, m = 7, 8
            kind, params = "rocksample", inputs.rocksample_params(n, m, 1, D=60)

            def prior(K, sd, n=n, m=m):
                return inputs.rocksample_belief(n, m, 1, K, 10_000 + sd % 100_003), inputs.weights(K)
        else:
            kind, params = "nav", inputs.nav_params(13, D=90)

            def prior(K, sd):
                return inputs.nav_belief(K, 10_000 + sd % 100_003, 13), inputs.weights(K)
        model = Model(kind, params)
        for budget in args.budgets:
            cfg = search_config(workers=args.workers, max_inflight=8 if args.workers > 1 else 1, max_batch=64,
                                batch_wait_us=200, time_budget_s=budget, xi=0.95, c_a=0.3, c_o=0.1)
            rets, steps, nodes, t_plan = [], [], [], []
            for ep in range(args.episodes):
                true_state = prior(1, 7_777 + ep)[0][:, 0]  # the world's state: a draw from the same prior
                t0 = time.perf_counter()
                log = online.run_episode(model, prior, true_state, K=args.K, steps=args.steps, config=cfg, seed=ep)
                dt = time.perf_counter() - t0
                rets.append(log["discounted_return"])
                steps.append(log["steps"])
                nodes.append(np.mean([s["nodes"] for s in log["search"]]))
                t_plan.append(dt / max(1, log["steps"]))
            print(json.dumps({"model": name, "budget_s": budget, "workers": args.workers, "K": args.K,
                              "episodes": args.episodes, "mean_discounted_return": float(np.mean(rets)),
                              "stderr": float(np.std(rets) / np.sqrt(len(rets))), "mean_steps": float(np.mean(steps)),
                              "mean_tree_nodes": float(np.mean(nodes)), "wall_s_per_step": float(np.mean(t_plan))}),
                  flush=True)
        model.close()


if __name__ == "__main__":
    main()
