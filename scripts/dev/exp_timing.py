"""Per-step device time of a batch with and without the library's K2 events,
in alternating order (diagnostic for bench.py)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import numpy as np
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import Model
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kind, params, st, w, seed, L = inputs.config_inputs(cfg)
m = Model(kind, params)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
if kind == "car":
    leaves = [(m.belief_load(a, b, c), -1, 0, 0) for a, b, c in inputs.car_roots(L, len(w))]
else:
    root = m.belief_load(st, w, seed)
    R = m.expand([(root, -1, 0, 0)])
    leaves = [(root, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], m.A, L)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
preps = {t: m.prepare(leaves, device_outputs=True, timing=t) for t in (False, "k2", True)}
def run(t, n=10, fl=True):
    ts = []
    for i in range(n):
        if fl: flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); steps, launches, nodes = m.run_prepared(preps[t], stream=s); e1.record(s)
        new = [nd for (lf, nd) in zip(leaves, nodes) if lf[1] >= 0]
        if new: m.node_release_many(new)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return np.median(ts), list(preps[t]["E"].phase_ms)
for t in (False, "k2", True): run(t, 3)
for rep in range(2):
    for t in (False, "k2", True, False):
        med, ph = run(t)
        print(f"cfg {cfg} timing={t}: median {med:.4f} ms  phases {[round(x,4) for x in ph]}", flush=True)
