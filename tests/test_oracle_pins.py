"""Pins of the CPU oracle against what the paper, SPEC.md and mathematics fix.

Every test here checks the oracle against something other than itself: known-
answer vectors, constants printed in the paper (tests/golden/), closed forms,
brute-force optimal values on tiny instances, and statistical event rates.
A plausible mistake in the oracle (a dropped term, a wrong sign or index, a
transposed operand) should fail at least one of them.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden_constants():
    out = {}
    with open(os.path.join(GOLDEN, "paper_constants.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            parts = line.split()
            out[parts[0]] = float(parts[1])
    return out


G = golden_constants()


# ----------------------------------------------------------------------------
# Philox4x32-10 (reading R13): third-party known-answer vectors
# ----------------------------------------------------------------------------
def test_philox_known_answers():
    n = 0
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            assert list(oracle.philox(v[0:4], v[4:6])) == v[6:10]
            n += 1
    assert n == 3


def test_thresholds_closed_form():
    for p in ("0.03", "0.01", "0.85", "0.1", "0.5"):
        assert oracle.threshold(float(p)) == int(G["T_" + p]) == math.floor(float(p) * 2**32)
    assert oracle.threshold(1.0) == 2**32  # p = 1: the event always fires
    assert oracle.threshold(0.0) == 0


# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------
def find_stream(model, s, a, t, seed, pred, max_ids=20000):
    """first scenario id whose step outcome satisfies pred(s2, z, r, term)"""
    for sid in range(max_ids):
        out = model.step(s, a, sid, t, seed)
        if pred(*out[:4]):
            return sid, out[:4]
    raise AssertionError("no stream found")


def rs_state(n, good_mask, cells):
    w1 = 0
    for r, (x, y) in enumerate(cells):
        w1 |= (0xFFFF if (x, y) == (-1, -1) else y * n + x) << (16 * r)
    return np.array([good_mask, w1], np.uint32)


# ----------------------------------------------------------------------------
# RockSample / MARS
# ----------------------------------------------------------------------------
def test_mars_action_counts_from_paper():
    for n, key in ((11, "mars_actions_11"), (15, "mars_actions_15"), (20, "mars_actions_20")):
        m = oracle.Model("rocksample", inputs.rocksample_params(n, n, 2))
        assert m.A == int(G[key])
    assert oracle.Model("rocksample", inputs.rocksample_params()).A == 13


def test_rs_sample_good_and_bad_rock():
    params = inputs.rocksample_params()  # RS(7,8), rock 0 at (2,0)
    m = oracle.Model("rocksample", params)
    s = rs_state(7, 0b1, [(2, 0)])
    s2, z, r, term, counted = m.step(s, 4, 0, 1, 5)
    assert r == G["rs_sample_good"] and s2[0] == 0 and not term and counted  # rock becomes bad
    s2b, _, r2, _, _ = m.step(s2, 4, 0, 2, 5)
    assert r2 == G["rs_sample_bad"] and s2b[0] == 0
    # sampling an empty cell: no reward, no effect (card)
    s3, _, r3, _, _ = m.step(rs_state(7, 0xFF, [(1, 1)]), 4, 0, 1, 5)
    assert r3 == 0.0 and s3[0] == 0xFF


def test_rs_exit_east_border_reward_and_terminal():
    m = oracle.Model("rocksample", inputs.rocksample_params())
    s2, z, r, term, _ = m.step(rs_state(7, 0, [(6, 4)]), 2, 0, 1, 9)
    assert r == G["rs_exit"] and term and z[0] == 3  # TERMINAL slot 3^R
    assert (s2[1] & 0xFFFF) == 0xFFFF
    # two robots: the world terminates only when both have exited
    m2 = oracle.Model("rocksample", inputs.rocksample_params(5, 2, 2))
    s2, z, r, term, _ = m2.step(rs_state(5, 0, [(4, 0), (1, 1)]), 2 + 7 * 0, 0, 1, 9)
    assert r == 10.0 and not term


def test_rs_sense_at_distance_zero_is_always_correct():
    m = oracle.Model("rocksample", inputs.rocksample_params())
    s_good = rs_state(7, 0b1, [(2, 0)])
    s_bad = rs_state(7, 0b0, [(2, 0)])
    for sid in range(2000):
        assert m.step(s_good, 5, sid, 1, 3)[1][0] == 1
        assert m.step(s_bad, 5, sid, 1, 3)[1][0] == 2


def test_rs_sense_accuracy_decays_with_distance():
    """accuracy 0.5 (1 + 2^(-d/d0)): far rock -> near coin flip"""
    m = oracle.Model("rocksample", inputs.rocksample_params())
    s = rs_state(7, 0xFF, [(0, 3)])  # rock 3 at (6,3): d = 6
    N = 20000
    correct = sum(m.step(s, 5 + 3, sid, 1, 11)[1][0] == 1 for sid in range(N))
    p = 0.5 * (1 + 2 ** (-6 / 4))
    assert abs(correct / N - p) < 5 * math.sqrt(p * (1 - p) / N)


def test_rs_upper_bound_all_bad_at_east_border():
    """all rocks bad, robot at the east border -> 10"""
    m = oracle.Model("rocksample", inputs.rocksample_params())
    assert m.upper(rs_state(7, 0, [(6, 5)])) == 10.0
    assert m.upper(rs_state(7, 0, [(-1, -1)])) == 0.0  # terminal


def test_rs_move_only_action_keeps_one_child():
    kind, params, st, w, seed, _ = inputs.config_inputs(2, K=60)
    m = oracle.Model(kind, params)
    root = m.belief_load(st, w, seed)
    o = m.expand([(root, -1, 0, 0)])
    for a in range(m.A):
        b0, b1 = a % 20, a // 20
        if b0 < 5 and b1 < 5:  # moves and samples on empty start cells
            nb = o["child_begin"][a + 1] - o["child_begin"][a]
            assert nb == 1 and o["child_count"][o["child_begin"][a]] == 60


def test_rs_always_east_rollout_closed_form():
    """Eq. 12 with an always-E default policy: 10 gamma^{n-1-x} exactly"""
    m = oracle.Model("rocksample", inputs.rocksample_params(extra="policy=east"))
    for x in range(7):
        s = rs_state(7, 0xFF, [(x, 2)])
        ret, ln, _, _ = m.rollout(s, None, 0, 0, 99)
        assert ln == 7 - x
        assert ret == pytest.approx(10 * 0.95 ** (6 - x), rel=1e-14)


# ----------------------------------------------------------------------------
# Navigation
# ----------------------------------------------------------------------------
def nav_model():
    return oracle.Model("nav", inputs.nav_params())


def nav_state(x, y, gate=0, occ_bits=0, words=5):
    s = np.zeros(words, np.uint32)
    s[0] = y * 13 + x + (gate << 8)
    s[1] = occ_bits
    return s


def test_nav_unknown_cells_match_state_space():
    assert inputs.nav_unknown_count() == int(G["nav_unknown_cells"])
    assert nav_model().SW == 1 + 124 // 32 + 1


def test_nav_rewards_from_paper():
    m = nav_model()
    s = nav_state(6, 0)
    _, _, r, term, _ = m.step(s, 0, 0, 1, 1)
    assert r == np.float32(G["nav_stay_reward"]) and not term
    # a successful move (find a stream without the 0.03 failure)
    sid, (s2, z, r, term) = find_stream(m, s, 5, 1, 1, lambda s2, z, r, t: (s2[0] & 0xFF) == 13 + 6)
    assert r == np.float32(G["nav_move_reward"])
    # crash into the wall row (known obstacle at (6,6)) leaves the position
    s = nav_state(6, 5)
    sid, (s2, z, r, term) = find_stream(m, s, 5, 1, 1, lambda s2, z, r, t: r == -1.0)
    assert r == G["nav_crash_reward"] and (s2[0] & 0xFF) == 5 * 13 + 6
    # goal (6,12) from (6,11): +20 and terminal
    s = nav_state(6, 11)
    sid, (s2, z, r, term) = find_stream(m, s, 5, 1, 1, lambda s2, z, r, t: t)
    assert r == G["nav_goal_reward"] and term and z[0] == 0x100


def test_nav_event_rates():
    """move failure 0.03, per-direction reading error 0.03, all eight readings
    correct w.p. 0.97^8"""
    m = nav_model()
    s = nav_state(6, 0)  # top row: N, NE, NW off-grid (occupied), others known free
    truth = 0b10000011  # bits N, NE, NW
    N = 20000
    fails = flips = allok = 0
    for sid in range(N):
        s2, z, r, term, _ = m.step(s, 7, sid, 3, 77)  # W: target (5,0) is free
        moved = (s2[0] & 0xFF) == 5
        fails += not moved
        if moved:
            true_bits = 0b10000011  # at (5,0): same geometry
            diff = int(z[0]) ^ true_bits
            flips += bin(diff).count("1")
            allok += diff == 0
    p = G["nav_move_fail"]
    assert abs(fails / N - p) < 5 * math.sqrt(p * (1 - p) / N)
    moved = N - fails
    q = G["nav_obs_flip"]
    assert abs(flips / (8 * moved) - q) < 5 * math.sqrt(q * (1 - q) / (8 * moved))
    pa = G["nav_all_correct"]
    assert abs(allok / moved - pa) < 5 * math.sqrt(pa * (1 - pa) / moved)
    assert truth == 0b10000011


def test_nav_rollout_one_step_to_horizon():
    """D - depth = 1 -> r + gamma * tail"""
    m = oracle.Model("nav", inputs.nav_params(D=5))
    s = nav_state(6, 0)
    ret, ln, _, _ = m.rollout(s, np.array([0], np.uint32), 3, 4, 21)
    # pi0 with t=4 even and z = all free picks S; find the step outcome independently
    s2, z, r, term, _ = m.step(s, 5, 3, 5, 21)
    assert ln == 1 and not term
    assert ret == pytest.approx(float(r) + 0.95 * m.tail, rel=1e-15)
    assert m.tail == pytest.approx(-0.2 / 0.05, rel=1e-7)


def test_nav_upper_bound_one_step_from_goal():
    m = nav_model()
    assert m.upper(nav_state(6, 11)) == 20.0  # S:66 reading: one move from the goal -> 20
    assert m.upper(nav_state(5, 11)) == 20.0  # diagonal
    assert m.upper(nav_state(6, 10)) == pytest.approx(20 * 0.95)


# ----------------------------------------------------------------------------
# Tiger -- closed forms
# ----------------------------------------------------------------------------
def test_tiger_listen_only_rollout_closed_form():
    m = oracle.Model("tiger", inputs.tiger_params(D=10))
    for side in (0, 1):
        ret, ln, _, _ = m.rollout(np.array([side], np.uint32), None, 5, 0, 3)
        assert ln == 10
        assert ret == pytest.approx(G["tiger_listen_rollout_D10"], abs=1e-12)
        assert ret == pytest.approx(-(1 - 0.95**10) / (1 - 0.95), abs=1e-12)


def test_tiger_open_correct_door_and_listen_accuracy():
    m = oracle.Model("tiger", inputs.tiger_params())
    s2, z, r, term, _ = m.step(np.array([0], np.uint32), 2, 0, 1, 1)  # tiger left, open right
    assert r == 10.0 and term and z[0] == 3
    _, _, r, _, _ = m.step(np.array([0], np.uint32), 1, 0, 1, 1)
    assert r == -100.0
    N = 20000
    ok = sum(m.step(np.array([1], np.uint32), 0, sid, 1, 4)[1][0] == 2 for sid in range(N))
    assert abs(ok / N - 0.85) < 5 * math.sqrt(0.85 * 0.15 / N)


def test_tiger_brute_force_depth_one_closed_form():
    """V*_1 = max(listen: -1 + gamma*0, open-left, open-right) for k tigers left of K"""
    for K, k in ((5, 2), (8, 8), (4, 0)):
        st = np.array([[0] * k + [1] * (K - k)], np.uint32)
        m = oracle.Model("tiger", inputs.tiger_params(D=1))
        root = m.belief_load(st, inputs.weights(K), 1)
        v = m.brute_force(root)
        pl = k / K
        expect = max(-1.0, pl * -100 + (1 - pl) * 10, (1 - pl) * -100 + pl * 10)
        assert v == pytest.approx(expect, abs=1e-6)


# ----------------------------------------------------------------------------
# Bounds: l <= V*_D <= u on tiny instances (north star invariant)
# ----------------------------------------------------------------------------
TINY = [
    ("tiger", inputs.tiger_params(D=5), 8),
    ("rocksample", "n=3 robots=1 D=4 gamma=0.95 rocks=1:0,2:2 starts=0:1", 4),
    ("rocksample", "n=3 robots=2 D=2 gamma=0.95 rocks=1:0 starts=0:0,0:2", 4),
    ("nav", inputs.nav_params(5, wall_y=2, gates=(1, 3), landmarks=[], goal=(2, 4), D=4), 3),
    ("car", inputs.car_params(peds=2, D=3), 4),
]


def tiny_belief(kind, params, K, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "tiger":
        return inputs.tiger_belief(K, seed)
    if kind == "rocksample":
        if "robots=1" in params:
            st = np.zeros((2, K), np.uint32)
            st[0] = rng.integers(0, 4, K)
            st[1] = 1 * 3 + 0
            return st
        st = np.zeros((2, K), np.uint32)
        st[0] = rng.integers(0, 2, K)
        st[1] = (0 * 3 + 0) | ((2 * 3 + 0) << 16)
        return st
    if kind == "nav":
        # 5x5: unknown cells are rows 1 and 3 (10 cells), occupied w.p. 0.1
        st = np.zeros((2, K), np.uint32)
        st[0] = rng.integers(0, 5, K) + (rng.integers(0, 2, K) << 8)
        occ = rng.random((K, 10)) < 0.1
        st[1] = (occ.astype(np.uint32) << np.arange(10, dtype=np.uint32)).sum(axis=1)
        return st
    # car 1 m before the goal at speed level 3, pedestrians next to the path
    st = inputs.car_belief(K, seed, peds=2)
    st[0] = np.float32(18.75).view(np.uint32)
    st[1] = 3
    st[4:] = np.array([19.75, 0.75, 20.0, -1.25], np.float32).view(np.uint32)[:, None]
    return st


@pytest.mark.parametrize("case", range(len(TINY)))
def test_bounds_bracket_brute_force_value(case):
    kind, params, K = TINY[case]
    m = oracle.Model(kind, params)
    for seed in (11, 12):
        st = tiny_belief(kind, params, K, seed)
        w = inputs.weights(K, seed, uniform=(seed % 2 == 1))
        root = m.belief_load(st, w, seed)
        o = m.expand([(root, -1, 0, 0)])
        q = m.brute_force_q(root)
        v = m.brute_force(root)
        assert v == pytest.approx(q.max(), abs=1e-12)
        tol = 1e-9
        # one-level Eq. 4 values bracket Q*_D(b, a)
        assert np.all(o["act_lower"] <= q + tol), (o["act_lower"], q)
        assert np.all(q <= o["act_upper"] + tol), (q, o["act_upper"])
        # children: l(b') <= V*_D(b') <= u(b')
        leaves = []
        for a in range(m.A):
            for c in range(o["child_begin"][a + 1] - o["child_begin"][a]):
                leaves.append((root, a, c, 1))
        o2 = m.expand(leaves, action_mask=np.zeros(m.A, np.uint8))
        for i, (_, a, c, _) in enumerate(leaves):
            ci = o["child_begin"][a] + c
            vc = m.brute_force(int(o2["node"][i]))
            assert o["child_lower"][ci] <= vc + tol
            assert vc <= o["child_upper"][ci] + tol
            assert o["child_lower"][ci] <= o["child_upper"][ci] + tol


# ----------------------------------------------------------------------------
# Grouping, Eq. 11 / Eq. 12 audits, update step, determinism
# ----------------------------------------------------------------------------
@pytest.fixture(scope="module", params=[1, 3, 4])
def expanded(request):
    cfg = request.param
    K = {1: 100, 3: 80, 4: 40}[cfg]
    kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=K, uniform=False, D={1: 20, 3: 30, 4: 25}[cfg])
    m = oracle.Model(kind, params)
    root = m.belief_load(st, w, seed)
    o = m.expand([(root, -1, 0, 0)], record=True)
    return m, root, o, st, w, seed


def test_children_partition_each_action(expanded):
    m, root, o, st, w, seed = expanded
    K = len(w)
    W = float(np.sum(w.astype(np.float64)))
    for a in range(m.A):
        b, e = o["child_begin"][a], o["child_begin"][a + 1]
        assert int(o["child_count"][b:e].sum()) == K  # sum N_c = |Phi_b|
        assert float(o["child_weight"][b:e].sum()) == pytest.approx(W, rel=1e-12)  # north star
        keys = {tuple(k) for k in o["child_obs"][b:e]}
        assert len(keys) == e - b
        # first-occurrence order: first ids strictly increasing
        assert np.all(np.diff(o["child_first"][b:e].astype(np.int64)) > 0)


def test_grouping_equals_dictionary_grouping(expanded):
    m, root, o, st, w, seed = expanded
    K = len(w)
    for a in range(m.A):
        rows = o["scen_obs"][a * K:(a + 1) * K]
        groups = {}
        for i, row in enumerate(rows):
            groups.setdefault(tuple(row), []).append(i)
        order = sorted(groups.values(), key=lambda g: g[0])
        b = o["child_begin"][a]
        assert len(order) == o["child_begin"][a + 1] - b
        for c, g in enumerate(order):
            assert o["child_count"][b + c] == len(g)
            assert o["child_first"][b + c] == g[0]  # root ids = positions
            assert list(o["scen_child"][a * K:(a + 1) * K][g]) == [c] * len(g)


def test_eq11_eq12_audit_by_independent_calls(expanded):
    """child u = weighted mean of u(s') recomputed by oracle_upper; child l =
    weighted mean of roll-outs recomputed by oracle_rollout"""
    m, root, o, st, w, seed = expanded
    K = len(w)
    ww = w.astype(np.float64)
    for a in range(0, m.A, max(1, m.A // 4)):
        sl = slice(a * K, (a + 1) * K)
        S2 = o["scen_states"][sl]
        Z = o["scen_obs"][sl]
        u = np.array([m.upper(s) for s in S2])  # 0 for terminal s'
        lam = np.zeros(K)
        for i in range(K):
            # a terminal s' gives return 0, length 0 and the FNV offset hash
            ret, ln, h, _ = m.rollout(S2[i], Z[i], i, 1, seed)
            lam[i] = ret
            assert ln == o["scen_len"][sl][i] and h == o["scen_hash"][sl][i]
            assert ret == o["scen_lower"][sl][i]
        np.testing.assert_allclose(o["scen_upper"][sl], u, rtol=0, atol=0)
        b, e = o["child_begin"][a], o["child_begin"][a + 1]
        ch = o["scen_child"][sl]
        for c in range(e - b):
            g = ch == c
            assert o["child_upper"][b + c] == pytest.approx(np.sum(ww[g] * u[g]) / np.sum(ww[g]), rel=1e-12, abs=1e-12)
            assert o["child_lower"][b + c] == pytest.approx(np.sum(ww[g] * lam[g]) / np.sum(ww[g]), rel=1e-12, abs=1e-12)
        # one-level Eq. 4
        r = o["scen_reward"][sl].astype(np.float64)
        W = ww.sum()
        assert o["act_reward"][a] == pytest.approx(np.sum(ww * r) / W, rel=1e-12, abs=1e-12)
        assert o["act_upper"][a] == pytest.approx(np.sum(ww * (r + m.gamma * u)) / W, rel=1e-12)
        assert o["act_lower"][a] == pytest.approx(np.sum(ww * (r + m.gamma * lam)) / W, rel=1e-12, abs=1e-12)


def test_update_step_equals_index_lists(expanded):
    """a1: the replay-filter arena equals the paper-style index list of the
    parent's scenarios that fell into the child"""
    m, root, o, st, w, seed = expanded
    K = len(w)
    leaves = []
    for a in range(m.A):
        for c in range(min(3, o["child_begin"][a + 1] - o["child_begin"][a])):
            leaves.append((root, a, c, 1))
    o2 = m.expand(leaves, action_mask=np.zeros(m.A, np.uint8))
    for i, (_, a, c, _) in enumerate(leaves):
        nd = m.node_read(int(o2["node"][i]))
        idx = np.nonzero(o["scen_child"][a * K:(a + 1) * K] == c)[0]
        assert list(nd["ids"]) == list(idx)
        np.testing.assert_array_equal(nd["w"], w[idx])
        np.testing.assert_array_equal(nd["states"].T, o["scen_states"][a * K:(a + 1) * K][idx])
        assert o2["n_scen"][i] == len(idx)


def test_determinism(expanded):
    m, root, o, st, w, seed = expanded
    o2 = m.expand([(root, -1, 0, 0)], record=True)
    for k in o:
        if isinstance(o[k], np.ndarray):
            np.testing.assert_array_equal(o[k], o2[k])


def test_terminal_start_rollout_and_all_terminal_node():
    """S:302 terminal start -> 0; S:295 all-terminal node -> zero future value"""
    m = oracle.Model("tiger", inputs.tiger_params())
    st = np.array([[2, 3, 2]], np.uint32)  # terminal states
    ret, ln, _, _ = m.rollout(st[:, 0], None, 0, 0, 1)
    assert ret == 0.0 and ln == 0
    root = m.belief_load(st, inputs.weights(3), 1)
    o = m.expand([(root, -1, 0, 0)])
    assert np.all(o["act_reward"] == 0) and np.all(o["act_upper"] == 0) and np.all(o["act_lower"] == 0)
    assert o["scenario_steps"] == 0
    assert np.all(o["child_count"] == 3)


# ----------------------------------------------------------------------------
# Driving -- invariants and closed-form single steps (the
# constants are PROPOSED: the paper defers the model to Bai 2015); the
# heading-noise statistics are pinned in test_oracle_pins_policy.py
# ----------------------------------------------------------------------------
def test_car_pedestrians_move_exactly_one_step_length():
    m = oracle.Model("car", inputs.car_params())
    assert m.A == int(G["car_actions"]) and m.elements == 21
    st = inputs.car_belief(16, 5)
    f = lambda wds: np.asarray(wds, np.uint32).view(np.float32)
    for k in range(16):
        s = st[:, k]
        s2, z, r, term, _ = m.step(s, 0, k, 1, 5)
        p0 = f(s[4:]).reshape(-1, 2).astype(np.float64)
        p1 = f(s2[4:]).reshape(-1, 2).astype(np.float64)
        d = np.linalg.norm(p1 - p0, axis=1)
        np.testing.assert_allclose(d, 0.25, atol=2e-6)


def test_car_failed_accelerate_keeps_speed_and_goals_unobserved():
    m = oracle.Model("car", inputs.car_params())
    s = inputs.car_belief(1, 5)[:, 0]
    sid, (s2, z, r, term) = find_stream(m, s, 1, 1, 5, lambda s2, z, r, t: (s2[1] & 0xFF) == 2)
    assert (s2[1] & 0xFF) == 2  # failed ACC: level unchanged
    N = 4000
    fails = sum((m.step(s, 1, i, 1, 6)[0][1] & 0xFF) == 2 for i in range(N))
    p = G["car_fail"]
    assert abs(fails / N - p) < 5 * math.sqrt(p * (1 - p) / N)
    # goals never appear in observations: observation words are position bins
    f = np.asarray(s2, np.uint32)[4:].view(np.float32).reshape(-1, 2)
    for i in range(20):
        bx, by = int(np.floor(2 * f[i, 0])), int(np.floor(2 * f[i, 1]))
        assert z[1 + i] == ((bx & 0xFFFF) | ((by & 0xFFFF) << 16))


def test_scenario_prefix_is_stable_across_K():
    """ids are global and the streams are keyed by (id, depth):
    the first K scenarios of a larger belief reproduce every per-scenario
    outcome of the K-scenario belief"""
    for cfg, D in ((2, 12), (3, 30)):
        kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=80, D=D)
        m = oracle.Model(kind, params)
        big = m.expand([(m.belief_load(st, inputs.weights(80), seed), -1, 0, 0)], record=True)
        small = m.expand([(m.belief_load(st[:, :50], inputs.weights(50), seed), -1, 0, 0)], record=True)
        for a in range(0, m.A, max(1, m.A // 7)):
            sb, ss = slice(a * 80, a * 80 + 50), slice(a * 50, a * 50 + 50)
            for k in ("scen_obs", "scen_reward", "scen_len", "scen_hash", "scen_states", "scen_upper", "scen_lower"):
                np.testing.assert_array_equal(big[k][sb], small[k][ss])


# Driving, closed-form single steps of card §3.4 on one pedestrian:
# goal and collision rewards, the speed clamp, u(s) at the goal line and at the
# start, pi0's gap rule, and a pedestrian's step direction toward its goal.
def _car1(xc, level, px, py, goal):
    s = np.zeros(6, np.uint32)
    s[0] = np.float32(xc).view(np.uint32)
    s[1] = level
    s[2] = goal
    s[4] = np.float32(px).view(np.uint32)
    s[5] = np.float32(py).view(np.uint32)
    return s


def _f(w):
    return float(np.uint32(w).view(np.float32))


CAR1 = "peds=1 D=90 gamma=0.95"


def test_car_reaching_the_goal_line_pays_100_and_ends():
    m = oracle.Model("car", CAR1)
    # v = 0.5 * level 2 = 1 m/s, dt 0.25 s: 19.9 -> 20.15 >= 20; pedestrian far
    # away at (2, -5) walking to (0, -10)
    for sid in range(8):
        s2, z, r, term, _ = m.step(_car1(19.9, 2, 2.0, -5.0, 0), 0, sid, 1, 3)
        assert term and z[0] == 0xFFFFFFFF and z[1] == 0
        assert abs(_f(s2[0]) - 20.15) < 1e-5
        assert abs(r - (-0.1 + 100.0)) < 1e-4
    # one step short of the line: only the time cost
    s2, z, r, term, _ = m.step(_car1(10.0, 2, 2.0, -5.0, 0), 0, 0, 1, 3)
    assert not term and abs(r + 0.1) < 1e-6
    assert (z[0] & 0xFFFF) == 20 + 0 and (z[0] >> 16) == 2  # floor(2 * 10.25), level 2


def test_car_collision_costs_speed_squared():
    m = oracle.Model("car", CAR1)
    # pedestrian on the car's path 0.25 m ahead of where the car lands: after
    # both move 0.25 m they are at most 0.5 m apart (< 1 m): collision
    for sid in range(8):
        s2, z, r, term, _ = m.step(_car1(5.0, 2, 5.5, 0.0, 1), 0, sid, 1, 3)
        assert term and z[0] == 0xFFFFFFFF
        assert abs(r - (-0.1 - 1000.0 * (1.0 ** 2 + 0.5))) < 1e-2
    # standing still (level 0, DEC clamps at 0) and braking: -0.1 - 0.1 - 1000 * 0.5
    s2, z, r, term, _ = m.step(_car1(5.0, 0, 5.3, 0.0, 1), 2, 0, 1, 3)
    assert term and (s2[1] & 0xFF) == 0
    assert abs(r - (-0.2 - 500.0)) < 1e-2


def test_car_speed_level_clamps_at_0_and_4():
    m = oracle.Model("car", CAR1)
    for sid in range(32):
        s2 = m.step(_car1(0.0, 4, 2.0, -5.0, 0), 1, sid, 1, 3)[0]
        assert (s2[1] & 0xFF) == 4 and abs(_f(s2[0]) - 0.5) < 1e-6  # v = 2 m/s
        s2 = m.step(_car1(0.0, 0, 2.0, -5.0, 0), 2, sid, 1, 3)[0]
        assert (s2[1] & 0xFF) == 0 and _f(s2[0]) == 0.0


def test_car_upper_bound_goal_line_and_start():
    m = oracle.Model("car", CAR1)
    g = 0.95
    assert abs(m.upper(_car1(19.5, 2, 2.0, -5.0, 0)) - 100.0) < 1e-9   # k = 1
    assert abs(m.upper(_car1(19.9, 2, 2.0, -5.0, 0)) - 100.0) < 1e-9   # k clamped to 1
    assert abs(m.upper(_car1(0.0, 2, 2.0, -5.0, 0)) - 100.0 * g ** 39) < 1e-9  # k = 40 half-metre bins
    t = _car1(0.0, 2, 2.0, -5.0, 0)
    t[1] |= 1 << 8
    assert m.upper(t) == 0.0


def test_car_default_policy_gap_rule():
    m = oracle.Model("car", CAR1)
    s = _car1(0.0, 2, 2.0, -5.0, 0)

    def z(cxb, pxb, pyb):
        return [(cxb & 0xFFFF) | (2 << 16), (pxb & 0xFFFF) | ((pyb & 0xFFFF) << 16)]

    assert m.default_action(s, z(10, 14, 0), 0, 1) == 2    # gap 4 <= 8: DECELERATE
    assert m.default_action(s, z(10, 18, -4), 0, 1) == 2   # gap 8, lowest lane bin
    assert m.default_action(s, z(10, 22, 3), 0, 1) == 0    # gap 12 <= 16: MAINTAIN
    assert m.default_action(s, z(10, 40, 0), 0, 1) == 1    # gap 30: ACCELERATE
    assert m.default_action(s, z(10, 9, 0), 0, 1) == 1     # behind the car
    assert m.default_action(s, z(10, 14, 4), 0, 1) == 1    # outside the lane (y >= 2 m)
    assert m.default_action(s, z(10, 14, -5), 0, 1) == 1   # outside the lane (y < -2 m)


def test_car_pedestrian_heads_to_its_goal_on_average():
    """The heading noise is symmetric about the goal direction: over
    many streams the mean step points at the goal, its length below 0.25 m."""
    m = oracle.Model("car", CAR1)
    goals = [(0.0, -10.0), (0.0, 10.0), (20.0, -10.0), (20.0, 10.0)]
    px, py = 10.0, 0.0
    for gi, (gx, gy) in enumerate(goals):
        d = np.zeros(2)
        N = 2000
        for sid in range(N):
            s2 = m.step(_car1(0.0, 0, px, py, gi), 0, sid, 1, 9)[0]
            d += (_f(s2[4]) - px, _f(s2[5]) - py)
        d /= N
        e = np.array([gx - px, gy - py]) / math.hypot(gx - px, gy - py)
        along, across = d @ e, d[0] * e[1] - d[1] * e[0]
        assert 0.15 < along < 0.25, (gi, along)
        assert abs(across) < 0.02, (gi, across)
    # a pedestrian standing on its goal stays there
    s2 = m.step(_car1(0.0, 0, 20.0, 10.0, 3), 0, 0, 1, 9)[0]
    assert (_f(s2[4]), _f(s2[5])) == (20.0, 10.0)


def test_mars_joint_sample_same_and_different_rocks():
    """Two robots (reading R19): a joint action is one sub-action
    per robot, |A| = (5 + m)^2; on the same good rock the first SAMPLE earns
    +10 and turns it bad, the second pays -10; on two good rocks +20."""
    rocks, _ = inputs.rocksample_layout(15, 15, 2, 7)
    m = oracle.Model("rocksample", inputs.rocksample_params(15, 15, 2))
    base = 5 + 15
    samp = 4 + base * 4
    (x0, y0), (x1, y1) = rocks[0], rocks[1]
    allgood = (1 << 15) - 1
    s2, z, r, term, _ = m.step(rs_state(15, allgood, [(x0, y0), (x0, y0)]), samp, 0, 1, 5)
    assert r == 0.0 and s2[0] == allgood & ~1 and not term
    s2, z, r, term, _ = m.step(rs_state(15, allgood, [(x0, y0), (x1, y1)]), samp, 0, 1, 5)
    assert r == 20.0 and s2[0] == allgood & ~0b11
    # the same rock bad: both pay -10
    s2, z, r, term, _ = m.step(rs_state(15, allgood & ~1, [(x0, y0), (x0, y0)]), samp, 0, 1, 5)
    assert r == -20.0
    # robot 0 exits east (+10) while robot 1 stays: not terminal; both
    # exit: terminal with +20
    east = 2
    s2, z, r, term, _ = m.step(rs_state(15, 0, [(14, 3), (5, 5)]), east + base * 0, 0, 1, 5)
    assert r == 10.0 and not term and (int(s2[1]) & 0xFFFF) == 0xFFFF
    s2, z, r, term, _ = m.step(rs_state(15, 0, [(14, 3), (14, 9)]), east + base * east, 0, 1, 5)
    assert r == 20.0 and term
