"""bench.py's timed loop in isolation, toggling the nvidia-smi clock sampler
(diagnostic)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import numpy as np
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import Model
import bench
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
prep = m.prepare(leaves, device_outputs=True, timing=False)
def loop(n=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    for i in range(n):
        flush.zero_()
        ev[i][0].record(s)
        steps, launches, nodes = m.run_prepared(prep, stream=s)
        ev[i][1].record(s)
        new = [nd for (lf, nd) in zip(leaves, nodes) if lf[1] >= 0]
        if new: m.node_release_many(new)
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in ev]))
for _ in range(3): m.run_prepared(prep, stream=s)
print("no sampler", loop(), flush=True)
clk = bench.ClockSampler(0).start(); time.sleep(0.3)
print("sampler", loop(), flush=True)
clk.stop()
print("sampler stopped", loop(), flush=True)
