"""Host-side profile of despot_plan on config 2 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200 import despot as D
kind, params, st, w, seed, _ = inputs.config_inputs(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
gm = D.Model(kind, params)
root = gm.belief_load(st, w, seed)
for W in (1, 8):
    c = D.search_config(workers=W, max_inflight=8 if W > 1 else 1, max_batch=64, batch_wait_us=300,
                        time_budget_s=1.0, xi=0.95, c_a=0.3, c_o=0.1)
    r = gm.plan(root, c)
    print(W, {k: r[k] for k in ("nodes", "expanded", "trials", "batches", "max_depth", "seconds")},
          "us/batch %.1f" % (1e6 * r["seconds"] / r["batches"]), "leaves/batch %.2f" % (r["expanded"] / r["batches"]),
          file=sys.stderr, flush=True)
