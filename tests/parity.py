"""Helpers comparing libdespot outputs with the oracle's.

Bar (BASELINE.json north star): discrete outputs bit-exact
(leaf sizes, CSR, child counts, first ids, observation keys, per-scenario
observations, rewards, roll-out lengths and action-sequence hashes, states);
values within 1e-5 relative, where "relative" is to max(|x_oracle|, M) and M
is the weighted mean of the absolute terms of that value (reading R12).
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import Model

RTOL = 1e-5


def close(g, o, M, what):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    M = np.broadcast_to(np.asarray(M, np.float64), o.shape)
    tol = RTOL * np.maximum(np.abs(o), M)
    bad = np.abs(g - o) > tol
    assert not bad.any(), f"{what}: {int(bad.sum())} values out of tolerance, e.g. gpu={g[bad][:4]} oracle={o[bad][:4]}"


def leaf_slices(out, A, L):
    cb = np.asarray(out["child_begin"], np.int64)
    return [[(int(cb[l * A + a]), int(cb[l * A + a + 1])) for a in range(A)] for l in range(L)]


def oracle_scales(om: oracle.Model, onode: int, O: dict, li: int, A: int, scen_base: int):
    """M for the values of oracle leaf li, from its per-scenario records."""
    nd = om.node_read(onode)
    w = nd["w"].astype(np.float64)
    n = len(w)
    W = w.sum()
    Ms = {}
    for a in range(A):
        sl = slice(scen_base + a * n, scen_base + (a + 1) * n)
        r = O["scen_reward"][sl].astype(np.float64)
        u = O["scen_upper"][sl]
        lam = O["scen_lower"][sl]
        ch = O["scen_child"][sl]
        Ms[("reward", a)] = np.sum(w * np.abs(r)) / W
        Ms[("upper", a)] = np.sum(w * np.abs(r + om.gamma * u)) / W
        Ms[("lower", a)] = np.sum(w * np.abs(r + om.gamma * lam)) / W
        nc = int(ch.max()) + 1 if n else 0
        mu, ml = np.zeros(nc), np.zeros(nc)
        for c in range(nc):
            g = ch == c
            mu[c] = np.sum(w[g] * np.abs(u[g])) / np.sum(w[g])
            ml[c] = np.sum(w[g] * np.abs(lam[g])) / np.sum(w[g])
        Ms[("cu", a)] = mu
        Ms[("cl", a)] = ml
    return Ms, n


def compare_batch(G, O, gm: Model, om: oracle.Model, pairs, check_scen=False):
    """pairs: list of (gpu leaf index, oracle leaf index).  O must come from a
    record=True oracle expansion of the oracle leaves (in order)."""
    A = gm.A
    gsl = leaf_slices(G, A, len(G["n_scen"]))
    osl = leaf_slices(O, A, len(O["n_scen"]))
    # oracle per-scenario base offsets
    obase = np.concatenate([[0], np.cumsum(np.asarray(O["n_scen"], np.int64) * A)])
    gbase = np.concatenate([[0], np.cumsum(np.asarray(G["n_scen"], np.int64) * A)])
    for gi, oi in pairs:
        assert int(G["n_scen"][gi]) == int(O["n_scen"][oi]), f"leaf {gi}: |Phi| differs"
        Ms, n = oracle_scales(om, int(O["node"][oi]), O, oi, A, int(obase[oi]))
        close(G["weight"][gi], O["weight"][oi], 0.0, "leaf weight")
        for a in range(A):
            gb, ge = gsl[gi][a]
            ob, oe = osl[oi][a]
            assert ge - gb == oe - ob, f"leaf {gi} action {a}: {ge - gb} vs {oe - ob} children"
            for k in ("child_count", "child_first"):
                assert np.array_equal(np.asarray(G[k][gb:ge], np.int64), np.asarray(O[k][ob:oe], np.int64)), \
                    f"leaf {gi} action {a}: {k}"
            assert np.array_equal(G["child_obs"][gb:ge], O["child_obs"][ob:oe]), f"leaf {gi} action {a}: keys"
            close(G["child_weight"][gb:ge], O["child_weight"][ob:oe], 0.0, "child weight")
            close(G["child_upper"][gb:ge], O["child_upper"][ob:oe], Ms[("cu", a)], "child upper (Eq. 11)")
            close(G["child_lower"][gb:ge], O["child_lower"][ob:oe], Ms[("cl", a)], "child lower (Eq. 12)")
            ga, oa = gi * A + a, oi * A + a
            close(G["act_reward"][ga], O["act_reward"][oa], Ms[("reward", a)], "r(b,a)")
            close(G["act_upper"][ga], O["act_upper"][oa], Ms[("upper", a)], "u(b,a) (Eq. 4)")
            close(G["act_lower"][ga], O["act_lower"][oa], Ms[("lower", a)], "l(b,a) (Eq. 4)")
        if check_scen:
            gs = slice(int(gbase[gi]), int(gbase[gi]) + A * n)
            os_ = slice(int(obase[oi]), int(obase[oi]) + A * n)
            assert np.array_equal(G["scen_obs"][gs], O["scen_obs"][os_]), "per-scenario observations"
            assert np.array_equal(G["scen_reward"][gs], O["scen_reward"][os_]), "per-scenario rewards"
            assert np.array_equal(G["scen_len"][gs], O["scen_len"][os_]), "roll-out lengths"
            assert np.array_equal(G["scen_hash"][gs].view(np.uint64), O["scen_hash"][os_]), "roll-out action hashes"
            assert np.array_equal(G["scen_states"][gs], O["scen_states"][os_]), "states after the step"
            if "scen_child" in G:  # each scenario's child ordinal
                assert np.array_equal(np.asarray(G["scen_child"][gs], np.int64),
                                      np.asarray(O["scen_child"][os_], np.int64)), "per-scenario child ordinals"
            # per-scenario returns: fp32 of the fp64 value
            lam = O["scen_lower"][os_]
            close(G["scen_lower"][gs], lam, np.abs(lam) + 1e-6, "per-scenario roll-out return")
            close(G["scen_upper"][gs], O["scen_upper"][os_], 0.0, "per-scenario u(s')")


def setup(cfg, K=None, L=None, uniform=True, D=None, gpu_flags=0):
    kind, params, st, w, seed, L = inputs.config_inputs(cfg, K=K, L=L, uniform=uniform, D=D)
    gm = Model(kind, params, flags=gpu_flags)
    om = oracle.Model(kind, params)
    return gm, om, st, w, seed, L


def expand_root_both(gm, om, st, w, seed, record=True):
    gr = gm.belief_load(st, w, seed)
    orr = om.belief_load(st, w, seed)
    G = gm.expand([(gr, -1, 0, 0)], record=record)
    O = om.expand([(orr, -1, 0, 0)], record=True)
    return gr, orr, G, O
