#!/usr/bin/env python3
"""Host-side trace of repeated expansion calls (DESPOT_HOST_TRACE=1 must be
set in the environment): configs 1 and 3, device and host outputs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1802_06215_b200 import inputs  # noqa: E402
from paper_1802_06215_b200.despot import Model  # noqa: E402

for cfg in (1, 3):
    kind, params, st, w, seed, L = inputs.config_inputs(cfg)
    m = Model(kind, params)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    root = m.belief_load(st, w, seed)
    R = m.expand([(root, -1, 0, 0)])
    leaves = [(root, -1, 0, 0)] if cfg == 1 else [(root, a, c, 1) for a, c in inputs.select_leaves(
        R["child_count"], R["child_begin"], m.A, L)]
    for dev in (True, False):
        prep = m.prepare(leaves, device_outputs=dev)
        for i in range(8):
            steps, launches, nodes = m.run_prepared(prep, stream=s)
            new = [n for (lf, n) in zip(leaves, nodes) if lf[1] >= 0]
            if new:
                m.node_release_many(new)
        print(f"--- config {cfg} device_outputs={dev} ---", file=sys.stderr, flush=True)
