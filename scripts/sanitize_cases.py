"""Small expansion batches that drive every family of kernels, for the
self-check runs (compute-sanitizer is closed on the GPU pool): run under the
self-check build (DESPOT_LIB=paper_1802_06215_b200/libdespot_checked.so,
device checks of index and protocol invariants) with --stress N, every case
runs N times and must return bit-identical outputs each time (a race in the
last-CTA finalize, the look-back scan, the merge or the atomics would show as
run-to-run differences), and every child array must be untouched past the
children the call reports (the binding zero-fills them: an out-of-range write
shows as a nonzero word).  Cases:

  fused     config 1 (RockSample(7,8) root): K2 + the finalize in K2's last CTA
  k1_dense  MARS(15,15) K=300, 12 depth-1 leaves: k1_update, K2, k3_count_grouped,
            k3_scan_lookback, k3_write_grouped
  rank      MARS with 3 robots' worth of slots is not a model, so navigation
            (257 slots): k3_rank_dense / k3_write_wide
  sparse    driving, 6 pedestrians, 4 roots: k2_car_*, k3_group_sparse, k3_write_sparse
  merge     driving scenario-sharded over 2 emulated ranks: k_pack_sparse, k3_merge_sparse,
            k1_update_sparse on the merged children
  exchange  the library-owned exchange at world 1 (DESPOT_MF_EXCHANGE): k4_* packing, its
            capacity retry, the sparse record round
  graph     a prepared batch (CUDA graph) and resident ones (DESPOT_X_RESIDENT: a root, and
            navigation's depth-1 leaves with the wide finalize restoring the scratch), three runs each

Usage: python scripts/sanitize_cases.py [--stress N] [CASE ...]   (no case: all)
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
    return [G, g.expand([(r, -1, 0, 0)], record=True)]


def k1_dense():
    kind, params, st, w, seed, L = inputs.config_inputs(2, K=300, L=12)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    R = g.expand([(r, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)
    return [R, g.expand([(r, a, c, 1) for a, c in lv]), g.expand([(r, a, c, 1) for a, c in lv[:3]], record=True)]


def rank():
    kind, params, st, w, seed, L = inputs.config_inputs(3, K=200, L=8, D=30)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    R = g.expand([(r, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)
    return [R, g.expand([(r, a, c, 1) for a, c in lv])]


def sparse():
    params = inputs.car_params(6, D=30)
    outs = []
    for flags in (1, 2, 4, 16):
        g = Model("car", params, flags=flags)
        roots = [g.belief_load(s, w_, sd) for s, w_, sd in inputs.car_roots(4, 64, peds=6)]
        outs.append(g.expand([(r, -1, 0, 0) for r in roots]))
    return outs


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
    return outs + run([[(rt[0], a, c, 1) for a, c in lv] for rt in roots])


def exchange():
    """the library-owned exchange (world 1 with DESPOT_MF_EXCHANGE): packed
    dense protocol (and its capacity retry), sparse record round"""
    import torch.distributed  # noqa: F401
    from paper_1802_06215_b200.despot import DESPOT_MF_EXCHANGE, Comm, comm_unique_id
    c = Comm(comm_unique_id(), 0, 1, 0)
    outs = []
    for extra in ("", " xratio16=1"):
        kind, params, st, w, seed, L = inputs.config_inputs(2, K=120, L=6)
        g = Model(kind, params + extra, flags=DESPOT_MF_EXCHANGE, comm=c)
        r = g.belief_load(st, w, seed)
        R = g.expand([(r, -1, 0, 0)])
        lv = inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)
        outs += [R, g.expand([(r, a, cc, 1) for a, cc in lv])]
    g = Model("car", inputs.car_params(6, D=30), flags=DESPOT_MF_EXCHANGE, comm=c)
    roots = [g.belief_load(s_, w_, sd) for s_, w_, sd in inputs.car_roots(3, 50, peds=6)]
    outs.append(g.expand([(r_, -1, 0, 0) for r_ in roots]))
    return outs


def graph():
    """prepared batches (CUDA graphs): repeated runs"""
    kind, params, st, w, seed, L = inputs.config_inputs(2, K=90, L=5)
    g = Model(kind, params)
    r = g.belief_load(st, w, seed)
    R = g.expand([(r, -1, 0, 0)])
    lv = [(r, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], g.A, L)]
    outs = []
    # a prepared batch of depth-1 leaves, and a resident one (self leaves: the
    # graph is K2 alone, its last CTA restores the scratch)
    kn, pn, stn, wn, sdn, Ln = inputs.config_inputs(3, K=150, L=8)
    gn = Model(kn, pn)
    rn = gn.belief_load(stn, wn, sdn)
    Rn = gn.expand([(rn, -1, 0, 0)])
    lvn = [(rn, a, c, 1) for a, c in inputs.select_leaves(Rn["child_count"], Rn["child_begin"], gn.A, Ln)]
    for g_, P in ((g, g.prepare(lv)), (g, g.prepare([(r, -1, 0, 0)], resident=True)),
                  (gn, gn.prepare(lvn, resident=True))):
        for _ in range(3):
            g_.run_prepared(P)
            o = {k: np.array(v, copy=True) for k, v in P["o"].items() if not k.startswith("_")}
            o.update({"_full_" + k: o[k] for k in ("child_count", "child_first", "child_weight", "child_upper",
                                                   "child_lower")})
            o["num_children"] = int(P["E"].num_children)
            outs.append(o)
    return outs


CASES = dict(fused=fused, k1_dense=k1_dense, rank=rank, sparse=sparse, merge=merge, exchange=exchange, graph=graph)

KEYS = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count", "child_first",
        "child_weight", "child_upper", "child_lower", "child_obs", "scen_obs", "scen_reward", "scen_upper",
        "scen_lower", "scen_len", "scen_hash", "scen_states")


def _untouched_tail(o, tag):
    """child arrays past the reported children are still the binding's zeros"""
    n = int(o.get("num_children", -1))
    if n < 0:
        return
    for k in ("child_count", "child_first", "child_weight", "child_upper", "child_lower"):
        full = o.get("_full_" + k)
        if full is not None:
            assert not np.any(np.asarray(full)[n:]), (tag, k, "write past num_children")


def _same(a, b, tag):
    for k in KEYS:
        if k in a:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (tag, k, "differs between runs")


if __name__ == "__main__":
    args = sys.argv[1:]
    stress = 1
    if args and args[0] == "--stress":
        stress, args = int(args[1]), args[2:]
    names = args or list(CASES)
    from paper_1802_06215_b200 import despot as _d
    print("library", _d.LIB_PATH, flush=True)
    for n in names:
        first = None
        for rep in range(stress):
            outs = CASES[n]()
            for j, o in enumerate(outs):
                _untouched_tail(o, (n, rep, j))
            if first is None:
                first = outs
            else:
                for j, (a, b) in enumerate(zip(first, outs)):
                    _same(a, b, (n, rep, j))
        print("case", n, "ok x", stress, flush=True)
