"""Per-call device time of a config-1 expansion under different timing forms,
with and without the L2 flush and the bench's nvidia-smi clock sampler
(diagnostic for bench.py's small-batch numbers)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import numpy as np
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import Model
import bench
kind, params, st, w, seed, L = inputs.config_inputs(1)
m = Model(kind, params)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
root = m.belief_load(st, w, seed)
leaves = [(root, -1, 0, 0)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for sampler in (False, True):
    clk = bench.ClockSampler(0).start() if sampler else None
    time.sleep(0.3)
    for timing in (False, "k2"):
        prep = m.prepare(leaves, device_outputs=True, timing=timing)
        for fl in (False, True):
            for _ in range(5): m.run_prepared(prep, stream=s)
            ts = []
            for i in range(30):
                if fl: flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s); m.run_prepared(prep, stream=s); e1.record(s)
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(f"sampler={sampler} timing={timing} flush={fl}: event ms median {np.median(ts):.4f} min {min(ts):.4f} max {max(ts):.4f}")
    if clk: clk.stop()
