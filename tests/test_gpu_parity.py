"""GPU parity: libdespot (through the C ABI) vs the CPU oracle on identical
seeded inputs.  Discrete outputs bit-exact, values within 1e-5 (parity.py)."""
import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import DespotError, Model

from parity import compare_batch, expand_root_both, setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


# ----------------------------------------------------------------------------
def test_stream_words_match_oracle_philox():
    gm = Model("tiger", inputs.tiger_params())
    rng = np.random.default_rng(3)
    ids = rng.integers(0, 2**31, 1000).astype(np.uint32)
    for seed, t, k in ((0, 0, 0), (0xDEADBEEF12345678, 7, 5), (1004, 90, 8), (2**64 - 1, 1, 3)):
        g = gm.stream_words(seed, ids, t, k)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        o = np.array([oracle.philox([i, t, k >> 2, 0], key)[k & 3] for i in ids], np.uint32)
        assert np.array_equal(g, o)


def test_k0_philox_ceiling_checksum_matches_oracle():
    """K0 draws the stream blocks (g, t) of every thread g and XOR-folds them:
    its checksum equals the oracle generator's over the same blocks."""
    gm = Model("tiger", inputs.tiger_params())
    for seed, n, blocks in ((1002, 1000, 3), (0xDEADBEEF12345678, 333, 7)):
        ms, cs = gm.philox_ceiling(seed, n, blocks, reps=2)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        x = 0
        for g in range(n):
            for t in range(1, blocks + 1):
                for v in oracle.philox([g, t, 0, 0], key):
                    x ^= int(v)
        assert cs == x and ms > 0.0
    with pytest.raises(DespotError):
        gm.philox_ceiling(1, 0, 1)


@pytest.mark.parametrize("cfg", [1, 3])
def test_expand_batch_bytes_bounds_the_outputs(cfg):
    """despot_expand_batch_bytes: the child bound equals the binding's and
    covers the children the call produces; the scenario bound covers the
    per-scenario records; the byte count matches the arrays' sizes."""
    gm, om, st, w, seed, L = setup(cfg, K=120 if cfg == 1 else 200, L=6)
    gr = gm.belief_load(st, w, seed)
    G0 = gm.expand([(gr, -1, 0, 0)])
    lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(G0["child_count"], G0["child_begin"], gm.A, L)]
    C, S, B = gm.batch_bytes(lv, record=True)
    assert C == gm.child_capacity_bound(lv)
    G = gm.expand(lv, record=True)
    assert int(G["child_begin"][-1]) <= C
    assert gm.A * int(np.sum(G["n_scen"])) <= S
    A, OW, SW, Lc = gm.A, gm.OW, gm.SW, len(lv)
    assert B == Lc * 16 + Lc * A * 12 + (Lc * A + 1) * 4 + C * (20 + 4 * OW) + S * (4 * OW + 24 + 4 * SW)
    with pytest.raises(DespotError):
        gm.batch_bytes([(123456789, 0, 0, 1)])
    gm.close()


# ----------------------------------------------------------------------------
# full configs (BASELINE.json), in the launch configuration bench.py times;
# the oracle checks a sample of the leaves (each leaf's outputs depend only on
# that leaf)
# ----------------------------------------------------------------------------
def _full_config(cfg, K=None, L=None, sample=(0, 1, -2, -1), action_mask=None):
    gm, om, st, w, seed, L = setup(cfg, K=K, L=L)
    gr, orr, G0, O0 = expand_root_both(gm, om, st, w, seed, record=False)
    compare_batch(G0, O0, gm, om, [(0, 0)])
    glv = inputs.select_leaves(G0["child_count"], G0["child_begin"], gm.A, L)
    olv = inputs.select_leaves(O0["child_count"], O0["child_begin"], om.A, L)
    assert glv == olv
    G = gm.expand([(gr, a, c, 1) for a, c in glv])
    idx = sorted({s % L for s in sample})
    O = om.expand([(orr, glv[i][0], glv[i][1], 1) for i in idx], record=True, action_mask=action_mask)
    if action_mask is None:
        compare_batch(G, O, gm, om, list(zip(idx, range(len(idx)))))
    else:
        # compare the masked actions only
        A = gm.A
        for j, i in enumerate(idx):
            assert int(G["n_scen"][i]) == int(O["n_scen"][j])
        acts = np.nonzero(action_mask)[0]
        for j, i in enumerate(idx):
            for a in acts:
                gb, ge = G["child_begin"][i * A + a], G["child_begin"][i * A + a + 1]
                ob, oe = O["child_begin"][j * A + a], O["child_begin"][j * A + a + 1]
                assert np.array_equal(G["child_first"][gb:ge], O["child_first"][ob:oe])
                assert np.array_equal(G["child_count"][gb:ge], O["child_count"][ob:oe])
                np.testing.assert_allclose(G["child_upper"][gb:ge], O["child_upper"][ob:oe], rtol=1e-5, atol=1e-5)
                np.testing.assert_allclose(G["child_lower"][gb:ge], O["child_lower"][ob:oe], rtol=1e-5, atol=1e-5)
                np.testing.assert_allclose(G["act_upper"][i * A + a], O["act_upper"][j * A + a], rtol=1e-5, atol=1e-5)
                np.testing.assert_allclose(G["act_lower"][i * A + a], O["act_lower"][j * A + a], rtol=1e-5, atol=1e-5)
    gm.close()


def test_config1_rocksample_root():
    gm, om, st, w, seed, L = setup(1)
    gr, orr, G, O = expand_root_both(gm, om, st, w, seed, record=True)
    compare_batch(G, O, gm, om, [(0, 0)], check_scen=True)
    assert G["scenario_steps"] == O["scenario_steps"]


def test_large_belief_few_slots_uses_warp_groups():
    """K2's warp-level observation groups (the LANE_RED = false form: many
    tiles per (leaf, action) and few slots per leaf, A * S < 1024): a
    RockSample(7,8) root with K = 2048 (64 tiles per action, 13 x 4 slots),
    its depth-1 children, and the record form, against the oracle; the timed
    and record kernels agree bit for bit."""
    gm, om, st, w, seed, L = setup(1, K=2048, uniform=False)
    gr, orr, G, O = expand_root_both(gm, om, st, w, seed, record=True)
    compare_batch(G, O, gm, om, [(0, 0)], check_scen=True)
    assert G["scenario_steps"] == O["scenario_steps"]
    _timed_form_equals_record(gm, [(gr, -1, 0, 0)], G)
    lv = inputs.select_leaves(G["child_count"], G["child_begin"], gm.A, 6)
    G1 = gm.expand([(gr, a, c, 1) for a, c in lv])
    O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    compare_batch(G1, O1, gm, om, [(i, i) for i in range(len(lv))])
    gm.close()


def test_config2_mars_64_leaves():
    _full_config(2)


def test_config3_nav_64_leaves():
    _full_config(3, sample=(0, 31, -1))


def _full_mars(n, m, K=500, L=64, sample=(0, 1, -2, -1)):
    """MARS(n, m) with two robots at BASELINE's config-2 batch shape (K = 500,
    64 depth-1 leaves): the paper's own instance MARS(20,20) with |A| = 625
     and MARS(11,11) with |A| = 256 -- other shared-memory
    table sizes, range masks and occupancies than the tested (15,15)."""
    params = inputs.rocksample_params(n, m, 2, D=20)
    seed = 1002
    st = inputs.rocksample_belief(n, m, 2, K, seed)
    w = inputs.weights(K, seed)
    gm, om = Model("rocksample", params), oracle.Model("rocksample", params)
    assert gm.A == (5 + m) ** 2
    gr, orr, G0, O0 = expand_root_both(gm, om, st, w, seed, record=False)
    compare_batch(G0, O0, gm, om, [(0, 0)])
    assert G0["scenario_steps"] == O0["scenario_steps"]
    glv = inputs.select_leaves(G0["child_count"], G0["child_begin"], gm.A, L)
    assert glv == inputs.select_leaves(O0["child_count"], O0["child_begin"], om.A, L)
    G = gm.expand([(gr, a, c, 1) for a, c in glv])
    idx = sorted({s % L for s in sample})
    O = om.expand([(orr, glv[i][0], glv[i][1], 1) for i in idx], record=True)
    compare_batch(G, O, gm, om, list(zip(idx, range(len(idx)))))
    # the timed form (prepared call, pinned host outputs) equals the plain call
    P = gm.prepare([(gr, a, c, 1) for a, c in glv], pinned=True)
    gm.run_prepared(P)
    for k in ("n_scen", "act_upper", "act_lower", "child_begin", "child_count", "child_first", "child_upper",
              "child_lower"):
        r = np.asarray(G[k]).reshape(-1)
        assert np.array_equal(np.asarray(P["o"][k])[: len(r)], r), k
    gm.close()


def test_mars_20_20_paper_instance_64_leaves():
    _full_mars(20, 20)


def test_mars_11_11_64_leaves():
    _full_mars(11, 11)


def test_nav_k5000_64_leaves():
    """Navigation at K = 5000 (the top of the paper's K sweep): 64
    depth-1 leaves, three sampled against the oracle."""
    _full_config(3, K=5000, sample=(0, 31, -1))


def test_config5_sweep_k4096_256_leaves():
    mask = np.zeros(400, np.uint8)
    mask[::17] = 1
    _full_config(5, K=4096, sample=(0, -1), action_mask=mask)


def test_config5_max_k32768_invariants_and_sampled_leaves():
    """The sweep's largest size (K = 32768, 256 leaves, the bench batch):
    invariants over every (leaf, action) -- the children partition the leaf
    (counts sum to |Phi|, weights to W), first ids strictly increase (first
    occurrence order), l <= u -- and two leaves against the oracle on a few
    actions (the oracle root expanded only for their actions)."""
    gm, om, st, w, seed, L = setup(5, K=32768)
    A = gm.A
    gr, orr = gm.belief_load(st, w, seed), om.belief_load(st, w, seed)
    G0 = gm.expand([(gr, -1, 0, 0)])
    glv = inputs.select_leaves(G0["child_count"], G0["child_begin"], A, L)
    G = gm.expand([(gr, a, c, 1) for a, c in glv])
    cb, cnt, first = G["child_begin"], G["child_count"], G["child_first"]
    for i in range(L):
        n = int(G["n_scen"][i])
        assert n == int(G0["child_count"][G0["child_begin"][glv[i][0]] + glv[i][1]])
        for a in range(A):
            b0, b1 = int(cb[i * A + a]), int(cb[i * A + a + 1])
            assert b1 > b0 and int(cnt[b0:b1].sum()) == n
            assert np.all(np.diff(first[b0:b1].astype(np.int64)) > 0)
            np.testing.assert_allclose(G["child_weight"][b0:b1].sum(), G["weight"][i], rtol=1e-5)
        assert np.all(G["act_lower"][i * A:(i + 1) * A] <= G["act_upper"][i * A:(i + 1) * A] + 1e-5)
    idx = [0, L - 1]
    mroot = np.zeros(A, np.uint8)
    for i in idx:
        mroot[glv[i][0]] = 1
    O0 = om.expand([(orr, -1, 0, 0)], action_mask=mroot)
    for i in idx:  # the same child under the same (action, ordinal) on both sides
        a, c = glv[i]
        assert int(O0["child_first"][O0["child_begin"][a] + c]) == int(G0["child_first"][G0["child_begin"][a] + c])
    mleaf = np.zeros(A, np.uint8)
    mleaf[::131] = 1
    O = om.expand([(orr, glv[i][0], glv[i][1], 1) for i in idx], action_mask=mleaf)
    for j, i in enumerate(idx):
        assert int(G["n_scen"][i]) == int(O["n_scen"][j])
        for a in np.nonzero(mleaf)[0]:
            gb, ge = G["child_begin"][i * A + a], G["child_begin"][i * A + a + 1]
            ob, oe = O["child_begin"][j * A + a], O["child_begin"][j * A + a + 1]
            assert np.array_equal(G["child_first"][gb:ge], O["child_first"][ob:oe])
            assert np.array_equal(G["child_count"][gb:ge], O["child_count"][ob:oe])
            np.testing.assert_allclose(G["child_upper"][gb:ge], O["child_upper"][ob:oe], rtol=1e-5, atol=1e-5)
            np.testing.assert_allclose(G["child_lower"][gb:ge], O["child_lower"][ob:oe], rtol=1e-5, atol=1e-5)
            np.testing.assert_allclose(G["act_upper"][i * A + a], O["act_upper"][j * A + a], rtol=1e-5, atol=1e-5)
            np.testing.assert_allclose(G["act_lower"][i * A + a], O["act_lower"][j * A + a], rtol=1e-5, atol=1e-5)
            np.testing.assert_allclose(G["act_reward"][i * A + a], O["act_reward"][j * A + a], rtol=1e-5, atol=1e-5)
    gm.close()


def test_max_leaves_per_batch():
    """kMaxLeaves = 4096 leaves in one batch (RockSample(7,8), K = 24): equal
    to the same leaves expanded in 8 batches of 512, and a batch of 4097 is
    refused."""
    gm, om, st, w, seed, _ = setup(1, K=24)
    gr = gm.belief_load(st, w, seed)
    R = gm.expand([(gr, -1, 0, 0)])
    pairs = [(a, c) for a in range(gm.A) for c in range(int(R["child_begin"][a + 1] - R["child_begin"][a]))]
    leaves = [(gr, a, c, 1) for a, c in (pairs * (4096 // len(pairs) + 1))[:4096]]
    big = gm.expand(leaves)
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_count", "child_first",
            "child_weight", "child_upper", "child_lower")
    parts = [gm.expand(leaves[k:k + 512]) for k in range(0, 4096, 512)]
    for k in keys:
        ref = np.concatenate([np.asarray(p[k]).reshape(-1) for p in parts])
        assert np.array_equal(np.asarray(big[k]).reshape(-1), ref), k
    gm.node_release_many([n for n in big["node"]] + [n for p in parts for n in p["node"]])
    with pytest.raises(DespotError):
        gm.expand(leaves + leaves[:1])


# ----------------------------------------------------------------------------
# small cases compared completely, incl. per-scenario records
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,K,L,uniform,D", [
    (1, 100, 6, False, 20),
    (2, 96, 16, False, 20),
    (2, 33, 5, True, 7),
    (3, 77, 9, False, 40),
    (3, 500, 3, True, 90),
])
def test_small_full_parity_with_records(cfg, K, L, uniform, D):
    gm, om, st, w, seed, _ = setup(cfg, K=K, L=L, uniform=uniform, D=D)
    gr, orr, G0, O0 = expand_root_both(gm, om, st, w, seed, record=True)
    compare_batch(G0, O0, gm, om, [(0, 0)], check_scen=True)
    assert G0["scenario_steps"] == O0["scenario_steps"]
    lv = inputs.select_leaves(G0["child_count"], G0["child_begin"], gm.A, L)
    G = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
    O = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    compare_batch(G, O, gm, om, [(i, i) for i in range(L)], check_scen=True)
    assert G["scenario_steps"] == O["scenario_steps"]
    # the update step (K1) materialises exactly the oracle's scenario subsets
    for i in range(L):
        gn, on = gm.node_read(G["node"][i]), om.node_read(int(O["node"][i]))
        assert np.array_equal(gn["ids"], on["ids"]) and np.array_equal(gn["states"], on["states"])
        assert np.array_equal(gn["w"], on["w"])
    # depth 2: children of the leaves
    lv2 = []
    for i in range(min(L, 3)):
        for a in range(0, gm.A, max(1, gm.A // 3)):
            b, e = G["child_begin"][i * gm.A + a], G["child_begin"][i * gm.A + a + 1]
            if e > b:
                lv2.append((i, a, int(e - b) - 1))
    G2 = gm.expand([(G["node"][i], a, c, 2) for i, a, c in lv2], record=True)
    O2 = om.expand([(int(O["node"][i]), a, c, 2) for i, a, c in lv2], record=True)
    compare_batch(G2, O2, gm, om, [(i, i) for i in range(len(lv2))], check_scen=True)
    gm.close()


def test_tiger_and_terminal_scenarios():
    gm = Model("tiger", inputs.tiger_params(D=12))
    om = oracle.Model("tiger", inputs.tiger_params(D=12))
    st = np.array([[0, 1, 2, 3, 1, 0, 3, 2, 1]], np.uint32)  # 2, 3 = terminal
    w = inputs.weights(9, 5, uniform=False)
    gr, orr = gm.belief_load(st, w, 77), om.belief_load(st, w, 77)
    G = gm.expand([(gr, -1, 0, 0)], record=True)
    O = om.expand([(orr, -1, 0, 0)], record=True)
    compare_batch(G, O, gm, om, [(0, 0)], check_scen=True)
    lv = [(a, c) for a in range(3) for c in range(int(G["child_begin"][a + 1] - G["child_begin"][a]))]
    G2 = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
    O2 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    compare_batch(G2, O2, gm, om, [(i, i) for i in range(len(lv))], check_scen=True)


def test_rocksample_terminal_and_ragged_beliefs():
    params = inputs.rocksample_params(5, 3, 2, D=9)
    gm, om = Model("rocksample", params), oracle.Model("rocksample", params)
    for K in (1, 31, 32, 33, 65):
        rng = np.random.default_rng(K)
        st = np.zeros((2, K), np.uint32)
        st[0] = rng.integers(0, 8, K)
        cells = rng.integers(0, 25, (K, 2))
        cells[rng.random((K, 2)) < 0.3] = 0xFFFF  # exited robots; both exited = terminal
        st[1] = cells[:, 0] | (cells[:, 1] << 16)
        w = inputs.weights(K, K, uniform=False)
        gr, orr = gm.belief_load(st, w, K), om.belief_load(st, w, K)
        G = gm.expand([(gr, -1, 0, 0)], record=True)
        O = om.expand([(orr, -1, 0, 0)], record=True)
        compare_batch(G, O, gm, om, [(0, 0)], check_scen=True)
        assert G["scenario_steps"] == O["scenario_steps"]


def test_mixed_beliefs_and_self_leaves_in_one_batch():
    kind, params, st, w, seed, _ = inputs.config_inputs(2, K=70)
    st2 = inputs.rocksample_belief(15, 15, 2, 50, 99)
    w2 = inputs.weights(50, 3, uniform=False)
    gm, om = Model(kind, params), oracle.Model(kind, params)
    ga, oa = gm.belief_load(st, w, seed), om.belief_load(st, w, seed)
    gb, ob = gm.belief_load(st2, w2, 4242), om.belief_load(st2, w2, 4242)
    G0 = gm.expand([(ga, -1, 0, 0), (gb, -1, 0, 0)])
    O0 = om.expand([(oa, -1, 0, 0), (ob, -1, 0, 0)], record=True)
    compare_batch(G0, O0, gm, om, [(0, 0), (1, 1)])
    leaves = [(ga, 7, 0, 1), (gb, 5 + 3, 1, 1), (ga, -1, 0, 0), (gb, 399, 0, 1)]
    oleaves = [(oa, 7, 0, 1), (ob, 5 + 3, 1, 1), (oa, -1, 0, 0), (ob, 399, 0, 1)]
    G = gm.expand(leaves)
    O = om.expand(oleaves, record=True)
    compare_batch(G, O, gm, om, [(i, i) for i in range(4)])


def test_errors_are_reported():
    kind, params, st, w, seed, _ = inputs.config_inputs(1)
    gm = Model(kind, params)
    gr = gm.belief_load(st, w, seed)
    with pytest.raises(DespotError) as e:
        gm.expand([(gr, 3, 0, 1)])  # parent not expanded yet
    assert e.value.code == -1
    gm.expand([(gr, -1, 0, 0)])
    with pytest.raises(DespotError) as e:
        gm.expand([(gr, 13, 0, 1)])
    assert e.value.code == -2  # EMODEL: action outside [-1, |A|)
    with pytest.raises(DespotError) as e:
        gm.expand([(gr, 0, 5, 1)])  # child ordinal 5 does not exist
    assert e.value.code == -1
    with pytest.raises(DespotError) as e:
        gm.expand([(gr, 0, 0, 2)])  # depth != parent depth + 1
    assert e.value.code == -1
    with pytest.raises(DespotError) as e:
        gm.expand([(gr, -1, 0, 0)], child_capacity=3)
    assert e.value.code == -4
    with pytest.raises(DespotError):
        gm.belief_load(st, np.zeros_like(w), seed)
    # the model still works after the errors
    G = gm.expand([(gr, 5, 0, 1)])
    assert G["n_scen"][0] > 0


def test_determinism_and_device_outputs():
    import torch
    gm, om, st, w, seed, L = setup(2, K=200, L=8)
    gr = gm.belief_load(st, w, seed)
    R = gm.expand([(gr, -1, 0, 0)])
    lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, L)]
    A1 = gm.expand(lv)
    A2 = gm.expand(lv)
    D1 = gm.expand(lv, device_outputs=True)
    torch.cuda.synchronize()
    for k in ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
              "child_first", "child_weight", "child_upper", "child_lower"):
        assert np.array_equal(A1[k], A2[k]), k  # exact reductions: bit-identical values
        d = D1[k].cpu().numpy()[: len(A1[k])]
        assert np.array_equal(d.view(A1[k].dtype) if d.dtype != A1[k].dtype else d, A1[k]), k


def test_fused_finalize_equals_separate_k3_and_prepared_calls():
    """Small dense batches finalize in K2's last CTA when expanded in one call
    (despot_expand_batch); the two-phase form (begin/end, world 1) runs the
    separate small K3.  Both, and the prepared-call binding, agree bit for bit."""
    import torch
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
            "child_first", "child_weight", "child_upper", "child_lower", "child_obs")
    for cfg, K, L in ((1, 100, 1), (2, 30, 4), (3, 31, 3)):
        gm, om, st, w, seed, _ = setup(cfg, K=K, L=L)
        gr = gm.belief_load(st, w, seed)
        R = gm.expand([(gr, -1, 0, 0)])
        lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, L)]
        for leaves in ([(gr, -1, 0, 0)], lv):
            F = gm.expand(leaves)
            b, _ = gm.expand_begin(leaves)
            U = gm.expand_end(b, leaves)
            prep = gm.prepare(leaves, device_outputs=False)
            steps, launches, nodes = gm.run_prepared(prep)
            torch.cuda.synchronize()
            # the fused batch skips the K3 launch (small S and L*A: the RockSample(7,8) case)
            assert F["launches"] < U["launches"] if cfg == 1 else F["launches"] <= U["launches"]
            assert F["scenario_steps"] == U["scenario_steps"] == steps
            for k in keys:
                assert np.array_equal(F[k], U[k]), (cfg, k)
                P = prep["o"][k]
                f = np.asarray(F[k]).reshape(-1)
                assert np.array_equal(np.asarray(P)[: len(f)], f), (cfg, k)
            for n in list(F["node"]) + list(U["node"]) + list(nodes):
                if n != gr:
                    gm.node_release(n)
        # the fused batch still matches the oracle
        orr = om.belief_load(st, w, seed)
        G = gm.expand([(gr, -1, 0, 0)])
        O = om.expand([(orr, -1, 0, 0)], record=True)
        compare_batch(G, O, gm, om, [(0, 0)])
        for n in G["node"]:
            if n != gr:
                gm.node_release(n)
        gm.close()


def test_pinned_host_outputs_equal_pageable():
    """Page-locked caller buffers take the direct-copy path (no staging): the
    results equal the pageable-buffer path bit for bit (dense and sparse)."""
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
            "child_first", "child_weight", "child_upper", "child_lower", "child_obs")
    gm, om, st, w, seed, L = setup(2, K=300, L=16)
    gr = gm.belief_load(st, w, seed)
    R = gm.expand([(gr, -1, 0, 0)])
    lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, L)]
    params = inputs.car_params(6, D=30)
    cm = Model("car", params)
    cl = [(cm.belief_load(s, w_, sd), -1, 0, 0) for s, w_, sd in inputs.car_roots(4, 60, peds=6)]
    for m, leaves in ((gm, lv), (gm, [(gr, -1, 0, 0)]), (cm, cl)):
        ref = m.expand(leaves)
        P = m.prepare(leaves, pinned=True)
        steps, launches, nodes = m.run_prepared(P)
        assert steps == ref["scenario_steps"]
        n = int(P["E"].num_children)
        assert n == ref["num_children"]
        for k in keys:
            a = np.asarray(P["o"][k])
            r = np.asarray(ref[k]).reshape(-1)
            assert np.array_equal(a[: len(r)], r), k
        m.node_release_many([nd for lf, nd in zip(leaves, ref["node"]) if lf[1] >= 0] +
                            [nd for lf, nd in zip(leaves, nodes) if lf[1] >= 0])


def test_rollout_bounds_match_oracle():
    for cfg in (1, 3):
        gm, om, st, w, seed, _ = setup(cfg, K=150, uniform=False)
        gr, orr = gm.belief_load(st, w, seed), om.belief_load(st, w, seed)
        gu, gl, pu, pl = gm.rollout_bounds(gr, per_scenario=True)
        ou, ol, qu, ql = om.rollout_bounds(orr, per_scenario=True)
        np.testing.assert_allclose(pu, qu, rtol=1e-6)
        np.testing.assert_allclose(pl, ql, rtol=1e-5, atol=1e-5 * np.abs(ql).max())
        assert abs(gu - ou) <= 1e-5 * abs(ou) and abs(gl - ol) <= 1e-5 * max(abs(ol), 1.0)


def test_fake_ranks_equal_single_gpu():
    """Scenario sharding with the ranks emulated one after the
    other on one GPU: the merged result equals world == 1 bit for bit."""
    import torch
    from paper_1802_06215_b200.dist import exchange_views
    kind, params, st, w, seed, L = inputs.config_inputs(2, K=300, L=12)
    g1 = Model(kind, params)
    r1 = g1.belief_load(st, w, seed)
    R = g1.expand([(r1, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g1.A, L)
    ref = g1.expand([(r1, a, c, 1) for a, c in lv])
    om = oracle.Model(kind, params)
    orr = om.belief_load(st, w, seed)
    O0 = om.expand([(orr, -1, 0, 0)], record=True)
    O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    for world in (2, 3, 4, 8):
        ms = [Model(kind, params, rank=r, world=world) for r in range(world)]
        roots = [m.belief_load(st, w, seed) for m in ms]

        def sharded(leaf_lists):
            begun = [m.expand_begin(ll) for m, ll in zip(ms, leaf_lists)]
            views = [exchange_views(ex, torch.device("cuda", 0)) for (_, ex) in begun]
            torch.cuda.synchronize()
            tot = sum(v[0] for v in views)
            mn = torch.stack([v[1] for v in views]).min(dim=0).values
            for s, mi in views:
                s.copy_(tot)
                mi.copy_(mn)
            torch.cuda.synchronize()
            return [m.expand_end(b, ll) for m, (b, _), ll in zip(ms, begun, leaf_lists)]

        outs0 = sharded([[(rt, -1, 0, 0)] for rt in roots])
        for o in outs0:
            for k in ("child_begin", "child_count", "child_first", "act_upper", "act_lower", "child_upper"):
                assert np.array_equal(o[k], R[k]), (world, k)
        outs = sharded([[(rt, a, c, 1) for a, c in lv] for rt in roots])
        for o in outs:
            for k in ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
                      "child_first", "child_weight", "child_upper", "child_lower", "child_obs"):
                assert np.array_equal(o[k], ref[k]), (world, k)
            assert o["scenario_steps"] == ref["scenario_steps"]
        # and against the oracle directly: every rank's merged result
        for o in outs0:
            compare_batch(o, O0, ms[0], om, [(0, 0)])
        for o in outs:
            compare_batch(o, O1, ms[0], om, [(i, i) for i in range(L)])
            assert o["scenario_steps"] == O1["scenario_steps"]


# ----------------------------------------------------------------------------
# driving (config 4): sparse 21-word keys, factored warp kernel
# ----------------------------------------------------------------------------
def _car_models(peds=20, D=90, grouped=False):
    params = inputs.car_params(peds, D=D)
    # forced factored (warp per scenario) -- or grouped (a lane group per
    # scenario, several scenarios per warp) -- and unfactored (thread per scenario)
    return (Model("car", params, flags=4 if grouped else 2), Model("car", params, flags=1),
            oracle.Model("car", params))


@pytest.mark.parametrize("grouped", [False, True])
def test_config4_car_64_roots_factored_and_unfactored(grouped):
    gw, gt, om = _car_models(grouped=grouped)
    roots = inputs.car_roots(64, 500)
    gws = [gw.belief_load(st, w, sd) for st, w, sd in roots]
    gts = [gt.belief_load(st, w, sd) for st, w, sd in roots]
    Gw = gw.expand([(r, -1, 0, 0) for r in gws])
    Gt = gt.expand([(r, -1, 0, 0) for r in gts])
    for k in ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
              "child_first", "child_weight", "child_upper", "child_lower", "child_obs"):
        assert np.array_equal(Gw[k], Gt[k]), k  # factored == unfactored, bit for bit
    assert Gw["scenario_steps"] == Gt["scenario_steps"]
    sample = [0, 17, 63]
    ors = [om.belief_load(*roots[j]) for j in sample]
    O = om.expand([(r, -1, 0, 0) for r in ors], record=True)
    compare_batch(Gw, O, gw, om, list(zip(sample, range(len(sample)))))


@pytest.mark.parametrize("peds,K,D,grouped", [(20, 64, 40, False), (6, 45, 90, False), (2, 7, 12, False),
                                               (12, 33, 30, False), (20, 64, 40, True), (3, 37, 25, True),
                                               (31, 20, 20, True)])
def test_car_small_full_parity_with_records(peds, K, D, grouped):
    gw, gt, om = _car_models(peds, D, grouped)
    st = inputs.car_belief(K, 5 + K, peds)
    st[0] = np.float32(12.0).view(np.uint32)  # closer to the goal: goal and collision outcomes occur
    w = inputs.weights(K, K, uniform=False)
    for gm in (gw, gt):
        gr, orr = gm.belief_load(st, w, 31), om.belief_load(st, w, 31)
        G0 = gm.expand([(gr, -1, 0, 0)], record=True)
        O0 = om.expand([(orr, -1, 0, 0)], record=True)
        compare_batch(G0, O0, gm, om, [(0, 0)], check_scen=True)
        assert G0["scenario_steps"] == O0["scenario_steps"]
        # depth-1 leaves through the full-key update step, then their expansion
        lv = [(a, c) for a in range(3) for c in range(min(3, int(G0["child_begin"][a + 1] - G0["child_begin"][a])))]
        G1 = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
        O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
        compare_batch(G1, O1, gm, om, [(i, i) for i in range(len(lv))], check_scen=True)
        assert G1["scenario_steps"] == O1["scenario_steps"]


def test_car_factored_equals_unfactored_1000_random_steps():
    """S:480 acceptance criterion 6: the factored step equals the unfactored
    step bit-exactly over 1000 random (s, a, phi, depth) triples -- here as
    1000 one-step expansions of random states (D = depth + 1, so the batch is
    exactly the step, its observation and its reward)."""
    rng = np.random.default_rng(6)
    for trial in range(10):
        peds = int(rng.choice([1, 6, 12, 20, 31]))
        gw, gt, _ = _car_models(peds, D=2, grouped=trial % 2 == 1)
        K = 100
        st = inputs.car_belief(K, trial, peds, layout_seed=trial)
        xs = rng.uniform(0, 20, K).astype(np.float32)
        st[0] = xs.view(np.uint32)
        st[1] = rng.integers(0, 5, K)
        for i in range(peds):
            st[4 + 2 * i] = rng.uniform(-2, 22, K).astype(np.float32).view(np.uint32)
            st[5 + 2 * i] = rng.uniform(-6, 6, K).astype(np.float32).view(np.uint32)
        w = inputs.weights(K)
        Gs = []
        for gm in (gw, gt):
            r = gm.belief_load(st, w, 1000 + trial)
            Gs.append(gm.expand([(r, -1, 0, 0)], record=True))
        for k in ("scen_obs", "scen_reward", "scen_states", "scen_len", "scen_hash", "scen_upper", "scen_lower"):
            assert np.array_equal(Gs[0][k], Gs[1][k]), (peds, k)


def test_concurrent_batches_from_host_threads():
    """The model is shared by many host threads (8 concurrent
    producers); every call uses its own scratch and stream and returns the
    same bits as a serial call."""
    import threading

    import torch
    gm, om, st, w, seed, L = setup(2, K=150, L=8)
    root = gm.belief_load(st, w, seed)
    R = gm.expand([(root, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, 24)
    jobs = [[(root, a, c, 1) for a, c in lv[i::8]] for i in range(8)]
    ref = [gm.expand(j) for j in jobs]
    got = [None] * 8
    errs = []

    def run(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    o = gm.expand(jobs[i], stream=s)
                    for n in o["node"]:
                        gm.node_release(n)
                got[i] = gm.expand(jobs[i], stream=s)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(8):
        for k in ("n_scen", "act_upper", "act_lower", "child_begin", "child_first", "child_upper", "child_lower"):
            assert np.array_equal(got[i][k], ref[i][k]), (i, k)


def test_sharded_model_rejects_record_and_single_call():
    kind, params, st, w, seed, _ = inputs.config_inputs(2, K=40)
    m = Model(kind, params, rank=0, world=2)
    r = m.belief_load(st, w, seed)
    assert m.node_info(r)[0] == 20  # ids 0, 2, 4, ... kept on rank 0 of 2
    with pytest.raises(DespotError):
        m.expand([(r, -1, 0, 0)])  # world > 1: begin / exchange / end only
    with pytest.raises(DespotError):
        m.expand_begin([(r, -1, 0, 0)], record=True)
    mc = Model("car", inputs.car_params(), rank=0, world=2)  # sparse keys shard too (two exchange rounds)
    rc = mc.belief_load(*inputs.car_roots(1, 30)[0])
    with pytest.raises(DespotError):
        mc.expand([(rc, -1, 0, 0)])


def _emulate_ranks(ms, leaf_lists):
    """The ranks of a sharded batch emulated one after the other on one GPU:
    every exchange round's SUM / MIN / MAX and all-gather done with torch."""
    import torch
    from paper_1802_06215_b200.dist import _CudaArray, round_views
    dev = torch.device("cuda", 0)
    begun = [m.expand_begin(ll) for m, ll in zip(ms, leaf_lists)]
    exs = [ex for _, ex in begun]
    W = len(ms)
    while True:
        views = [round_views(ex, dev) for ex in exs]
        torch.cuda.synchronize()
        for key in ("sums", "mins", "maxs"):
            vs = [v[key] for v in views]
            if vs[0] is None:
                continue
            s = torch.stack(vs)
            red = s.sum(0) if key == "sums" else s.min(0).values if key == "mins" else s.max(0).values
            for v in vs:
                v.copy_(red)
        if views[0]["gather"] is not None:
            blk = views[0]["gather"][1]
            assert all(v["gather"][1] == blk for v in views)  # identical block size on every rank
            bufs = [torch.as_tensor(_CudaArray(v["gather"][0], W * blk, "|u1"), device=dev) for v in views]
            for r in range(W):
                for q in range(W):
                    if q != r:
                        bufs[q][r * blk:(r + 1) * blk].copy_(bufs[r][r * blk:(r + 1) * blk])
        torch.cuda.synchronize()
        if not exs[0].more:
            assert not any(ex.more for ex in exs)
            break
        exs = [m.batch_exchange(b) for m, (b, _) in zip(ms, begun)]
    cap = 4 * max(m.child_capacity_bound(ll) for m, ll in zip(ms, leaf_lists))  # filtered nodes: see the bound
    return [m.expand_end(b, ll, child_capacity=cap) for m, (b, _), ll in zip(ms, begun, leaf_lists)]


def test_car_sharded_equals_single_gpu():
    """Driving (sparse 21-word keys) scenario-sharded over 2/3/4 emulated ranks:
    local grouping, MAX round, record all-gather, exact-key merge -- equal to
    world == 1 bit for bit, for 6 roots and for depth-1 children (K1 filters
    by the merged global child keys)."""
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
            "child_first", "child_weight", "child_upper", "child_lower", "child_obs")
    params = inputs.car_params(6, D=30)
    croots = inputs.car_roots(6, 80, peds=6)
    g1 = Model("car", params)
    r1 = [g1.belief_load(s, w_, sd) for s, w_, sd in croots]
    ref0 = g1.expand([(r, -1, 0, 0) for r in r1])
    R = g1.expand([(r1[0], -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], g1.A, 5)
    ref1 = g1.expand([(r1[0], a, c, 1) for a, c in lv])

    def same(o, ref, tag):
        for k in keys:
            assert np.array_equal(o[k], ref[k]), (tag, k)
        assert o["scenario_steps"] == ref["scenario_steps"], tag

    om = oracle.Model("car", params)
    ors = [om.belief_load(s, w_, sd) for s, w_, sd in croots]
    O0 = om.expand([(r, -1, 0, 0) for r in ors], record=True)
    O1 = om.expand([(ors[0], a, c, 1) for a, c in lv], record=True)
    for world in (2, 3, 4):
        ms = [Model("car", params, rank=r, world=world) for r in range(world)]
        roots = [[m.belief_load(s, w_, sd) for s, w_, sd in croots] for m in ms]
        for o in _emulate_ranks(ms, [[(r, -1, 0, 0) for r in rt] for rt in roots]):
            same(o, ref0, (world, "roots"))
            compare_batch(o, O0, ms[0], om, [(i, i) for i in range(len(croots))])  # and the oracle directly
        for o in _emulate_ranks(ms, [[(rt[0], -1, 0, 0)] for rt in roots]):
            same(o, R, (world, "root 0"))
        for o in _emulate_ranks(ms, [[(rt[0], a, c, 1) for a, c in lv] for rt in roots]):
            same(o, ref1, (world, "children"))
            compare_batch(o, O1, ms[0], om, [(i, i) for i in range(len(lv))])
            assert o["scenario_steps"] == O1["scenario_steps"]


def test_gpu_scenario_prefix_is_stable_across_K():
    kind, params, st, w, seed, _ = inputs.config_inputs(2, K=80, D=12)
    gm = Model(kind, params)
    big = gm.expand([(gm.belief_load(st, inputs.weights(80), seed), -1, 0, 0)], record=True)
    small = gm.expand([(gm.belief_load(st[:, :50], inputs.weights(50), seed), -1, 0, 0)], record=True)
    for a in range(0, gm.A, 13):
        sb, ss = slice(a * 80, a * 80 + 50), slice(a * 50, a * 50 + 50)
        for k in ("scen_obs", "scen_reward", "scen_len", "scen_hash", "scen_states", "scen_upper", "scen_lower"):
            assert np.array_equal(big[k][sb], small[k][ss]), k


AGG_KEYS = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count", "child_first",
            "child_weight", "child_upper", "child_lower", "child_obs")


def _timed_form_equals_record(gm, leaves, Grec):
    """The same leaves through the timed kernels (record=False: UNI_SEED round
    keys, the dynamic tile grid, the finalize fused into K2's last CTA or the
    grouped / wide / sparse K3 variants) give the record run's aggregates bit
    for bit -- and so the oracle's."""
    G = gm.expand(leaves)
    for k in AGG_KEYS:
        assert np.array_equal(np.asarray(G[k]), np.asarray(Grec[k])), k
    assert G["scenario_steps"] == Grec["scenario_steps"]
    gm.node_release_many([n for lf, n in zip(leaves, G["node"]) if lf[1] >= 0])


def _car_edge_belief(K, peds=2):
    """Hand-placed driving states (card §3.4): the goal line one step away,
    a pedestrian on the car's path, speed levels 0 and 4, a pedestrian
    standing on its goal (the d2 < 1e-6 branch), a terminal scenario, a
    pedestrian on or next to the edges of pi0's lane test (y = +-2, x on a
    car bin boundary)."""
    rng = np.random.Generator(np.random.PCG64(11))
    st = np.zeros((4 + 2 * peds, K), np.uint32)
    goals_xy = [(0.0, -10.0), (0.0, 10.0), (20.0, -10.0), (20.0, 10.0)]
    f = lambda v: np.float32(v).view(np.uint32)
    for k in range(K):
        case = k % 6
        xc = [19.9, 5.0, 0.0, 19.76, 12.0, 3.0][case]
        level = [2, 2, 0, 4, 1, 3][case]
        g = rng.integers(0, 4, size=peds)
        st[0, k], st[1, k] = f(xc), level | ((1 << 8) if (case == 5 and k % 12 == 5) else 0)
        st[2, k] = int(sum(int(g[i]) << (2 * i) for i in range(min(peds, 16))))
        for i in range(peds):
            if i == 0 and case == 1:
                x, y = xc + 0.6, 0.1 * (k % 3)          # on the car's path
            elif i == 0 and case == 2:
                x, y = goals_xy[g[i]]                  # on its own goal
            elif i == 1 and case in (3, 4):            # near pi0's lane edges, ahead of the car
                x = xc + 0.5 * rng.integers(-1, 16) + (0.0 if k % 4 else 0.01 * rng.random())
                y = float(rng.choice([-2.0, 2.0])) + float(rng.choice([0.0, 0.02, -0.02, 0.13, -0.13]))
            else:
                x, y = 2.0 + 17.0 * rng.random(), -5.0 + 10.0 * rng.random()
            st[4 + 2 * i, k], st[5 + 2 * i, k] = f(x), f(y)
    return st


def test_car_coordinates_beyond_the_bins_rejected():
    """belief_load refuses driving coordinates outside +-4096 m or not finite
    (the int16 observation bins, reading R21); 4096 itself is accepted"""
    gm = Model("car", inputs.car_params(2, D=20), flags=1)
    K = 4
    w = inputs.weights(K, 5)
    for word, bad in ((0, 4097.0), (4, -5000.0), (7, np.inf), (5, np.nan)):
        st = _car_edge_belief(K, 2)
        st[word, 1] = np.float32(bad).view(np.uint32)
        with pytest.raises(DespotError):
            gm.belief_load(st, w, 3)
    st = _car_edge_belief(K, 2)
    st[4, 2] = np.float32(4096.0).view(np.uint32)
    gm.node_release(gm.belief_load(st, w, 3))
    gm.close()


@pytest.mark.parametrize("grouped", [False, True])
def test_car_edge_states_match_oracle(grouped):
    peds, K = 2, 47
    gw, gt, om = _car_models(peds, 20, grouped)
    st = _car_edge_belief(K, peds)
    w = inputs.weights(K, K, uniform=False)
    for gm in (gw, gt):
        gr, orr = gm.belief_load(st, w, 77), om.belief_load(st, w, 77)
        G0 = gm.expand([(gr, -1, 0, 0)], record=True)
        O0 = om.expand([(orr, -1, 0, 0)], record=True)
        compare_batch(G0, O0, gm, om, [(0, 0)], check_scen=True)
        assert G0["scenario_steps"] == O0["scenario_steps"]
        _timed_form_equals_record(gm, [(gr, -1, 0, 0)], G0)
        lv = [(a, c) for a in range(3) for c in range(min(4, int(G0["child_begin"][a + 1] - G0["child_begin"][a])))]
        G1 = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
        O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
        compare_batch(G1, O1, gm, om, [(i, i) for i in range(len(lv))], check_scen=True)
        assert G1["scenario_steps"] == O1["scenario_steps"]
        _timed_form_equals_record(gm, [(gr, a, c, 1) for a, c in lv], G1)


# ----------------------------------------------------------------------------
# navigation edge states (card §3.3): next to the goal, on the gate cells, in
# the corners, fully blocked and fully free unknown maps, terminal scenarios;
# the 13x13 map and smaller maps (other state word counts)
# ----------------------------------------------------------------------------
def _nav_edge_belief(K, n, wall_y, gates, goal, landmarks, seed):
    nu = inputs.nav_unknown_count(n, wall_y, landmarks)
    st = inputs.nav_belief(K, seed, n, wall_y, landmarks, p_occ=0.1)
    gx, gy = goal
    cells = [(gx, gy - 1), (gx - 1, gy), (gates[0], wall_y), (gates[1], wall_y), (0, 0), (n - 1, n - 1),
             (n - 1, 0), (0, n - 1), (gx, gy - 2)]
    for k in range(K):
        x, y = cells[k % len(cells)]
        gate = (k // len(cells)) & 1
        st[0, k] = (y * n + x) | (gate << 8) | ((1 << 9) if k % 17 == 16 else 0)
        if k % 5 == 3:    # every unknown cell occupied
            for b in range(nu):
                st[1 + b // 32, k] |= np.uint32(1 << (b % 32))
        elif k % 5 == 4:  # every unknown cell free
            st[1:, k] = 0
    return st


@pytest.mark.parametrize("n,wall_y,gates,goal,landmarks,K,D", [
    (13, None, (3, 9), None, None, 61, 90),
    (5, 2, (1, 3), (2, 4), [], 33, 30),
    (9, 4, (2, 6), (4, 8), [(1, 2), (7, 6)], 40, 50),
])
def test_nav_edge_states_match_oracle(n, wall_y, gates, goal, landmarks, K, D):
    params = inputs.nav_params(n, wall_y=wall_y, gates=gates, landmarks=landmarks, goal=goal, D=D)
    wy = n // 2 if wall_y is None else wall_y
    gl = (n // 2, n - 1) if goal is None else goal
    lm = inputs.NAV_LANDMARKS_13 if landmarks is None else landmarks
    gm, om = Model("nav", params), oracle.Model("nav", params)
    st = _nav_edge_belief(K, n, wy, gates, gl, lm, K)
    w = inputs.weights(K, K + 1, uniform=False)
    gr, orr = gm.belief_load(st, w, 5 + K), om.belief_load(st, w, 5 + K)
    G0 = gm.expand([(gr, -1, 0, 0)], record=True)
    O0 = om.expand([(orr, -1, 0, 0)], record=True)
    compare_batch(G0, O0, gm, om, [(0, 0)], check_scen=True)
    assert G0["scenario_steps"] == O0["scenario_steps"]
    _timed_form_equals_record(gm, [(gr, -1, 0, 0)], G0)
    lv = [(a, c) for a in range(gm.A) for c in range(min(2, int(G0["child_begin"][a + 1] - G0["child_begin"][a])))]
    G1 = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
    O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    compare_batch(G1, O1, gm, om, [(i, i) for i in range(len(lv))], check_scen=True)
    assert G1["scenario_steps"] == O1["scenario_steps"]
    _timed_form_equals_record(gm, [(gr, a, c, 1) for a, c in lv], G1)
    gm.close()


def test_mars_edge_states_match_oracle():
    """MARS(15,15), 2 robots (card §3.2): robots standing on rocks (both on
    the same rock too), on the east border, one robot exited, all rocks good
    or all bad; a leaf's expansion plus depth-1 leaves against the oracle."""
    n, m, R = 15, 15, 2
    params = inputs.rocksample_params(n, m, R)
    rocks, starts = inputs.rocksample_layout(n, m, R, 7)
    gm, om = Model("rocksample", params), oracle.Model("rocksample", params)
    K = 70
    rng = np.random.default_rng(3)
    st = np.zeros((2, K), np.uint32)
    for k in range(K):
        case = k % 7
        good = [(1 << m) - 1, 0, int(rng.integers(0, 1 << m))][k % 3]
        j0, j1 = int(rng.integers(0, m)), int(rng.integers(0, m))
        c = {0: [rocks[j0], rocks[j0]], 1: [rocks[j0], rocks[j1]], 2: [(n - 1, 3), (n - 1, 11)],
             3: [(-1, -1), rocks[j1]], 4: [rocks[j0], (-1, -1)], 5: [(n - 1, 0), starts[1]],
             6: [starts[0], starts[1]]}[case]
        st[0, k] = good
        st[1, k] = sum((0xFFFF if xy == (-1, -1) else xy[1] * n + xy[0]) << (16 * r) for r, xy in enumerate(c))
    w = inputs.weights(K, 9, uniform=False)
    gr, orr = gm.belief_load(st, w, 123), om.belief_load(st, w, 123)
    G0 = gm.expand([(gr, -1, 0, 0)], record=True)
    O0 = om.expand([(orr, -1, 0, 0)], record=True)
    compare_batch(G0, O0, gm, om, [(0, 0)], check_scen=True)
    assert G0["scenario_steps"] == O0["scenario_steps"]
    _timed_form_equals_record(gm, [(gr, -1, 0, 0)], G0)
    lv = [(a, int(G0["child_begin"][a + 1] - G0["child_begin"][a]) - 1) for a in range(0, gm.A, 23)]
    G1 = gm.expand([(gr, a, c, 1) for a, c in lv], record=True)
    O1 = om.expand([(orr, a, c, 1) for a, c in lv], record=True)
    compare_batch(G1, O1, gm, om, [(i, i) for i in range(len(lv))], check_scen=True)
    assert G1["scenario_steps"] == O1["scenario_steps"]
    _timed_form_equals_record(gm, [(gr, a, c, 1) for a, c in lv], G1)
    gm.close()


def test_prepared_graph_runs_equal_plain_calls():
    """despot_batch_prepare / despot_batch_run (one CUDA graph per repeated
    batch): every run equals the plain call bit for bit, returns new nodes
    (distinct handles, usable as parents of the next batch), for dense and
    sparse keys, roots and depth-1 leaves, host and device outputs; a run whose
    parent was released fails cleanly."""
    import torch
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
            "child_first", "child_weight", "child_upper", "child_lower", "child_obs")
    for cfg, K, L in ((1, 100, 1), (2, 150, 12), (3, 120, 6)):
        gm, om, st, w, seed, _ = setup(cfg, K=K, L=L)
        gr = gm.belief_load(st, w, seed)
        R = gm.expand([(gr, -1, 0, 0)])
        lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, L)]
        for leaves in ([(gr, -1, 0, 0)], lv):
            ref = gm.expand(leaves)
            for dev, res in ((False, False), (True, False), (True, True), (False, True)):
                P = gm.prepare(leaves, device_outputs=dev, pinned=not dev, resident=res)
                assert P["graph"] is not None
                seen = set()
                for run in range(3):
                    steps, launches, nodes = gm.run_prepared(P)
                    torch.cuda.synchronize()
                    assert steps == ref["scenario_steps"]
                    for k in keys:
                        r = np.asarray(ref[k]).reshape(-1)
                        got = P["o"][k]
                        got = got.cpu().numpy() if dev else np.asarray(got)
                        got = got.reshape(-1)[: len(r)]
                        assert np.array_equal(got.view(r.dtype) if got.dtype != r.dtype else got, r), (cfg, k, run)
                    new = [int(n) for lf, n in zip(leaves, nodes) if lf[1] >= 0]
                    assert not (set(new) & seen)
                    seen |= set(new)
                    if new and run == 2:  # a prepared run's node is a parent like any other
                        G2 = gm.expand([(new[0], 0, 0, 2)])
                        assert G2["n_scen"][0] > 0
        gm.close()
    # sparse keys (driving roots)
    params = inputs.car_params(6, D=30)
    cm = Model("car", params)
    cl = [(cm.belief_load(s, w_, sd), -1, 0, 0) for s, w_, sd in inputs.car_roots(4, 60, peds=6)]
    ref = cm.expand(cl)
    P = cm.prepare(cl, pinned=True)
    for run in range(2):
        cm.run_prepared(P)
        for k in keys:
            r = np.asarray(ref[k]).reshape(-1)
            assert np.array_equal(np.asarray(P["o"][k]).reshape(-1)[: len(r)], r), k
    # a released parent
    gm, om, st, w, seed, _ = setup(2, K=60, L=2)
    gr = gm.belief_load(st, w, seed)
    R = gm.expand([(gr, -1, 0, 0)])
    lv = [(gr, a, c, 1) for a, c in inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, 2)]
    G1 = gm.expand(lv)
    leaves2 = [(G1["node"][0], 3, 0, 2)]
    P = gm.prepare(leaves2)
    gm.run_prepared(P)
    gm.node_release(G1["node"][0])
    with pytest.raises(DespotError):
        gm.run_prepared(P)
    gm.close()


def test_resident_prepared_batches():
    """DESPOT_X_RESIDENT (the scratch restored by K2's last CTA -- fused
    finalize -- or by the wide finalize's CTAs, the status in mapped host
    memory; self leaves: the graph is K2 alone): many runs equal the plain
    call and the oracle -- several roots of two beliefs, Tiger with terminal
    scenarios, RockSample(7,8), depth-1 leaves of RockSample and navigation --
    and after a
    failed run (child capacity too small) the next prepared run of the model
    is still exact; a failed resident batch sets up again and fails the same
    way (no state left over from the failed run)."""
    import torch
    keys = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count",
            "child_first", "child_weight", "child_upper", "child_lower", "child_obs")

    def check(gm, om, leaves, oleaves, runs=6):
        ref = gm.expand(leaves)
        O = om.expand(oleaves, record=True)
        compare_batch(ref, O, gm, om, [(i, i) for i in range(len(leaves))])
        for dev in (True, False):
            P = gm.prepare(leaves, device_outputs=dev, pinned=not dev, resident=True)
            for run in range(runs):
                steps, _, _ = gm.run_prepared(P)
                torch.cuda.synchronize()
                assert steps == ref["scenario_steps"], run
                assert int(P["E"].num_children) == ref["num_children"]
                for k in keys:
                    r = np.asarray(ref[k]).reshape(-1)
                    got = P["o"][k]
                    got = (got.cpu().numpy() if dev else np.asarray(got)).reshape(-1)[: len(r)]
                    assert np.array_equal(got.view(r.dtype) if got.dtype != r.dtype else got, r), (k, run, dev)

    gm, om, st, w, seed, _ = setup(1, K=100)
    roots = [(gm.belief_load(st, w, seed), -1, 0, 0), (gm.belief_load(st[:, :37], w[:37], seed + 5), -1, 0, 0)]
    oroots = [(om.belief_load(st, w, seed), -1, 0, 0), (om.belief_load(st[:, :37], w[:37], seed + 5), -1, 0, 0)]
    check(gm, om, roots[:1], oroots[:1])
    check(gm, om, roots, oroots)
    # a failing resident batch: too small a child capacity, twice (set up again), then a good one
    bad = gm.prepare(roots[:1], device_outputs=True, resident=True, child_capacity=1)
    for _ in range(2):
        with pytest.raises(DespotError):
            gm.run_prepared(bad)
    check(gm, om, roots[:1], oroots[:1], runs=2)
    gm.close()
    # depth-1 leaves (new arenas every run): the fused finalize (RockSample,
    # a few leaves) and navigation's wide finalize, whose CTAs restore their
    # own slots and whose last CTA publishes the status
    for cfg, K, L in ((1, 100, 5), (3, 120, 6), (3, 300, 24)):
        gm, om, st, w, seed, _ = setup(cfg, K=K, L=L)
        gr, orr = gm.belief_load(st, w, seed), om.belief_load(st, w, seed)
        R = gm.expand([(gr, -1, 0, 0)])
        om.expand([(orr, -1, 0, 0)])
        lv = inputs.select_leaves(R["child_count"], R["child_begin"], gm.A, L)
        check(gm, om, [(gr, a, c, 1) for a, c in lv], [(orr, a, c, 1) for a, c in lv], runs=4)
        gm.close()
    tm = Model("tiger", inputs.tiger_params(D=12))
    to = oracle.Model("tiger", inputs.tiger_params(D=12))
    tst = np.array([[0, 1, 2, 3, 1, 0, 3, 2, 1]], np.uint32)  # 2, 3 = terminal
    tw = inputs.weights(9, 5, uniform=False)
    check(tm, to, [(tm.belief_load(tst, tw, 77), -1, 0, 0)], [(to.belief_load(tst, tw, 77), -1, 0, 0)])
    tm.close()


@pytest.mark.parametrize("peds,K,D", [(20, 48, 40), (6, 40, 30), (31, 20, 20), (12, 33, 30), (3, 37, 25)])
def test_car_paired_lanes_equal_thread_kernel_and_oracle(peds, K, D):
    """DESPOT_MF_PAIRED (a lane pair per scenario, each lane owning half of a
    step's Philox blocks) is bit-identical to the thread-per-scenario kernel
    (roots and depth-1 leaves, per-scenario records) and matches the oracle."""
    from paper_1802_06215_b200.despot import DESPOT_MF_PAIRED
    params = inputs.car_params(peds, D=D)
    gp, gt, om = Model("car", params, flags=DESPOT_MF_PAIRED), Model("car", params, flags=1), oracle.Model("car", params)
    st = inputs.car_belief(K, 9 + K, peds)
    st[0] = np.float32(12.0).view(np.uint32)
    w = inputs.weights(K, K, uniform=False)
    rp, rt, ro = gp.belief_load(st, w, 31), gt.belief_load(st, w, 31), om.belief_load(st, w, 31)
    for rec in (True, False):
        P0 = gp.expand([(rp, -1, 0, 0)], record=rec)
        T0 = gt.expand([(rt, -1, 0, 0)], record=rec)
        for k in AGG_KEYS + (("scen_obs", "scen_reward", "scen_states", "scen_len", "scen_hash", "scen_upper",
                              "scen_lower") if rec else ()):
            assert np.array_equal(np.asarray(P0[k]), np.asarray(T0[k])), (rec, k)
    O0 = om.expand([(ro, -1, 0, 0)], record=True)
    compare_batch(P0, O0, gp, om, [(0, 0)])
    lv = [(a, c) for a in range(3) for c in range(min(3, int(P0["child_begin"][a + 1] - P0["child_begin"][a])))]
    P1 = gp.expand([(rp, a, c, 1) for a, c in lv], record=True)
    O1 = om.expand([(ro, a, c, 1) for a, c in lv], record=True)
    compare_batch(P1, O1, gp, om, [(i, i) for i in range(len(lv))], check_scen=True)


@pytest.mark.parametrize("cfg,K,L", [(2, 120, 10), (3, 90, 8), (1, 100, 6)])
def test_host_index_lists_equal_replay_filter(cfg, K, L):
    """The paper's update form: the host receives every
    scenario's child ordinal (RECORD's scen_child, equal to the oracle's) and
    builds each leaf's index list of parent positions; expanding the leaves
    from those lists (DESPOT_X_INDEX_LISTS: gather + replay) gives the nodes
    and outputs of the replay + filter form bit for bit.  A list naming a
    scenario of another child is refused (EINVAL)."""
    gm, om, st, w, seed, _ = setup(cfg, K=K, L=L)
    gr, orr, G0, O0 = expand_root_both(gm, om, st, w, seed, record=True)
    n = int(G0["n_scen"][0])
    assert np.array_equal(np.asarray(G0["scen_child"], np.int64), np.asarray(O0["scen_child"], np.int64))
    lv = inputs.select_leaves(G0["child_count"], G0["child_begin"], gm.A, L)
    lists = [np.nonzero(np.asarray(G0["scen_child"][a * n:(a + 1) * n]) == c)[0] for a, c in lv]
    ref = gm.expand([(gr, a, c, 1) for a, c in lv])
    got = gm.expand([(gr, a, c, 1) for a, c in lv], index_lists=lists)
    for k in AGG_KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    # the update replays only the listed scenarios (replay + filter replays every parent scenario)
    assert 0 < got["scenario_steps"] <= ref["scenario_steps"]
    for i in range(L):
        a_, b_ = gm.node_read(got["node"][i]), gm.node_read(ref["node"][i])
        assert np.array_equal(a_["ids"], b_["ids"]) and np.array_equal(a_["states"], b_["states"])
    # a list holding a scenario of another child of the same action
    a, c = lv[0]
    other = np.nonzero(np.asarray(G0["scen_child"][a * n:(a + 1) * n]) != c)[0]
    if len(other):
        bad = sorted(set(lists[0].tolist()) | {int(other[0])})
        with pytest.raises(DespotError) as e:
            gm.expand([(gr, a, c, 1)], index_lists=[bad])
        assert e.value.code == -1
    with pytest.raises(DespotError):
        gm.expand([(gr, a, c, 1)], index_lists=[[n + 5]])  # outside the parent
    gm.close()


def test_torch_allocator_hooks():
    """despot_opts' allocator hooks with torch's caching allocator: the same
    results as the library's own stream-ordered allocations (roots, depth-1
    leaves, a prepared graph batch); the node arenas live in torch's pool and
    go back to it when released."""
    import torch
    kind, params, st, w, seed, L = inputs.config_inputs(2, K=150, L=8)
    plain, hooked = Model(kind, params), Model(kind, params, allocator="torch")
    before = torch.cuda.memory_allocated()
    rp, rh = plain.belief_load(st, w, seed), hooked.belief_load(st, w, seed)
    assert torch.cuda.memory_allocated() > before  # the hooked root arena came from torch
    P0, H0 = plain.expand([(rp, -1, 0, 0)]), hooked.expand([(rh, -1, 0, 0)])
    lv = inputs.select_leaves(P0["child_count"], P0["child_begin"], plain.A, L)
    P1 = plain.expand([(rp, a, c, 1) for a, c in lv])
    H1 = hooked.expand([(rh, a, c, 1) for a, c in lv])
    for k in AGG_KEYS:
        assert np.array_equal(np.asarray(P1[k]), np.asarray(H1[k])), k
    mid = torch.cuda.memory_allocated()
    hooked.node_release_many(H1["node"])
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() < mid  # released arenas went back to torch's pool
    prep = hooked.prepare([(rh, a, c, 1) for a, c in lv])
    hooked.run_prepared(prep)
    for k in AGG_KEYS:
        r = np.asarray(P1[k]).reshape(-1)
        assert np.array_equal(np.asarray(prep["o"][k]).reshape(-1)[: len(r)], r), k
    hooked.close()
    plain.close()
