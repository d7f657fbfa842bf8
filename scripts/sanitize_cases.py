"""Small expansion batches for compute-sanitizer (memcheck / racecheck /
synccheck).  Each case drives one family of kernels at a size the sanitizer
finishes in seconds:

  fused     config 1 (RockSample(7,8) root): K2 + the finalize in K2's last CTA
  k1_dense  MARS(15,15) K=300, 12 depth-1 leaves: k1_update, K2, k3_count_grouped,
            k3_scan_lookback, k3_write_grouped
  rank      MARS with 3 robots' worth of slots is not a model, so navigation
            (257 slots): k3_rank_dense / k3_write_wide
  sparse    driving, 6 pedestrians, 4 roots: k2_car_*, k3_group_sparse, k3_write_sparse
  merge     driving scenario-sharded over 2 emulated ranks: k_pack_sparse, k3_merge_sparse,
            k1_update_sparse on the merged children

Usage: python scripts/sanitize_cases.py CASE [CASE ...]   (no case: all)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1802_06215_b200 import inputs  # noqa: E402
from paper_1802_06215_b200.despot import Model  # noqa: E402


def fused():
    kind, params, st, w, seed, _ = inputs.config_inputs(1)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    G = g.expand([(r, -1, 0, 0)])
    assert G["num_children"] > 0
    G = g.expand([(r, -1, 0, 0)], record=True)


def k1_dense():
    kind, params, st, w, seed, L = inputs.config_inputs(2, K=300, L=12)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    R = g.expand([(r, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)
    g.expand([(r, a, c, 1) for a, c in lv])
    g.expand([(r, a, c, 1) for a, c in lv[:3]], record=True)


def rank():
    kind, params, st, w, seed, L = inputs.config_inputs(3, K=200, L=8, D=30)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    R = g.expand([(r, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)
    g.expand([(r, a, c, 1) for a, c in lv])


def sparse():
    params = inputs.car_params(6, D=30)
    for flags in (1, 2, 4):
        g = Model("car", params, flags=flags)
        roots = [g.belief_load(s, w_, sd) for s, w_, sd in inputs.car_roots(4, 64, peds=6)]
        g.expand([(r, -1, 0, 0) for r in roots])


def merge():
    import torch
    from paper_1802_06215_b200.dist import round_views, _CudaArray
    params = inputs.car_params(6, D=30)
    croots = inputs.car_roots(3, 64, peds=6)
    world = 2
    ms = [Model("car", params, rank=r, world=world) for r in range(world)]
    roots = [[m.belief_load(s, w_, sd) for s, w_, sd in croots] for m in ms]
    dev = torch.device("cuda", 0)

    def run(leaf_lists):
        begun = [m.expand_begin(ll) for m, ll in zip(ms, leaf_lists)]
        exs = [ex for (_, ex) in begun]
        while True:
            vs = [round_views(ex, dev) for ex in exs]
            torch.cuda.synchronize()
            for key, op in (("sums", "sum"), ("mins", "min"), ("maxs", "max")):
                if vs[0][key] is None:
                    continue
                st = torch.stack([v[key] for v in vs])
                red = st.sum(0) if op == "sum" else st.min(0).values if op == "min" else st.max(0).values
                for v in vs:
                    v[key].copy_(red)
            if vs[0]["gather"] is not None:
                blk = vs[0]["gather"][1]
                bufs = [torch.as_tensor(_CudaArray(v["gather"][0], world * blk, "|u1"), device=dev) for v in vs]
                for r in range(world):
                    for b in bufs:
                        if b.data_ptr() != bufs[r].data_ptr():
                            b[r * blk:(r + 1) * blk].copy_(bufs[r][r * blk:(r + 1) * blk])
            torch.cuda.synchronize()
            if not exs[0].more:
                break
            exs = [m.batch_exchange(b) for m, (b, _) in zip(ms, begun)]
        return [m.expand_end(b, ll) for m, (b, _), ll in zip(ms, begun, leaf_lists)]

    outs = run([[(r, -1, 0, 0) for r in rt] for rt in roots])
    assert np.array_equal(outs[0]["child_first"], outs[1]["child_first"])
    o = outs[0]
    lv = inputs.select_leaves(o["child_count"], o["child_begin"], ms[0].A, 4)
    run([[(rt[0], a, c, 1) for a, c in lv] for rt in roots])


CASES = dict(fused=fused, k1_dense=k1_dense, rank=rank, sparse=sparse, merge=merge)

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case", n, "ok", flush=True)
