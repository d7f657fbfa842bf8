"""despot_plan: the host tree driver on libdespot's GPU backend."""
import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import Model, search_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def test_plan_converges_to_brute_force_on_gpu():
    st = np.array([[0, 1, 1, 0, 1, 1, 0, 1]], np.uint32)
    w = inputs.weights(8)
    params = inputs.tiger_params(D=4)
    gm, om = Model("tiger", params), oracle.Model("tiger", params)
    gr, orr = gm.belief_load(st, w, 5), om.belief_load(st, w, 5)
    res = gm.plan(gr, workers=1, max_inflight=1, max_batch=1, max_trials=2000, xi=0.5)
    v = om.brute_force(orr)
    assert abs(res["root_lower"] - v) < 1e-4 and abs(res["root_upper"] - v) < 1e-4, (res, v)
    assert res["action"] == int(np.argmax(om.brute_force_q(orr)))


@pytest.mark.parametrize("cfg", [2, 3])
def test_parallel_plan_batches_leaves(cfg):
    kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=200)
    gm = Model(kind, params)
    root = gm.belief_load(st, w, seed)
    u0, l0 = gm.rollout_bounds(root)
    res = gm.plan(root, workers=8, max_inflight=8, max_batch=64, batch_wait_us=500, time_budget_s=0.5, xi=0.95,
                  c_a=0.3, c_o=0.1)
    assert res["expanded"] > 1 and res["batches"] >= 1 and res["trials"] > 0
    assert res["expanded"] / res["batches"] > 1.5  # leaves of many trials per launch
    assert res["root_lower"] <= res["root_upper"] + 1e-4
    assert res["root_upper"] <= u0 + 1e-4 and res["root_lower"] >= l0 - 1e-4
    # the root node survives the search; its children arenas were released
    n, d = gm.node_info(root)
    assert n == 200 and d == 0


# ----------------------------------------------------------------------------
# closed loop (NEXT-4): world step and particle-filter update through libdespot
# ----------------------------------------------------------------------------
def test_world_step_and_belief_update_match_the_oracle():
    from paper_1802_06215_b200 import online
    kind, params, st, w, seed, _ = inputs.config_inputs(1, K=60)
    gm, om = Model(kind, params), oracle.Model(kind, params)
    rng = np.random.default_rng(3)
    for trial in range(6):
        s = st[:, rng.integers(0, st.shape[1])]
        a = int(rng.integers(0, gm.A))
        s2, z, r, term = online.world_step(gm, s, a, 77 + trial)
        # the same one-scenario belief on the oracle
        orr = om.belief_load(s.reshape(-1, 1), np.ones(1, np.float32), 77 + trial)
        O = om.expand([(orr, -1, 0, 0)], record=True)
        c0 = int(O["child_begin"][a])
        assert np.array_equal(np.asarray(O["child_obs"]).reshape(-1, gm.OW)[c0], z)
        assert abs(float(O["act_reward"][a]) - r) <= 1e-6 * max(1.0, abs(r))
        oc = om.expand([(orr, a, 0, 1)], record=True)
        assert np.array_equal(om.node_read(oc["node"][0])["states"][:, 0], s2)
    # particle-filter update: the child (a, z) of a belief, GPU == oracle
    gr, orr = gm.belief_load(st, w, seed), om.belief_load(st, w, seed)
    O = om.expand([(orr, -1, 0, 0)], record=True)
    for a in (0, 5, 9):
        c0, c1 = int(O["child_begin"][a]), int(O["child_begin"][a + 1])
        for c in range(c0, c1):
            z = np.asarray(O["child_obs"]).reshape(-1, gm.OW)[c]
            upd = online.belief_update(gm, gr, a, z)
            assert upd is not None
            oc = om.expand([(orr, a, c - c0, 1)], record=True)
            ref = om.node_read(oc["node"][0])
            assert np.array_equal(upd[0], ref["states"]) and np.array_equal(upd[1], ref["w"])
    # an observation no particle produced: deprivation
    assert online.belief_update(gm, gr, 0, np.array([0xFFFF], np.uint32)) is None


def test_closed_loop_episode_is_deterministic():
    from paper_1802_06215_b200 import online
    kind, params, st, w, seed, _ = inputs.config_inputs(1, K=100)

    def prior(K, sd):
        return inputs.rocksample_belief(7, 8, 1, K, 1000 + sd % 997), inputs.weights(K)

    true_state = st[:, 7]
    cfg = search_config(workers=1, max_inflight=1, max_batch=1, max_trials=60, xi=0.95, c_a=0.3)
    runs = []
    for _ in range(2):
        gm = Model(kind, params)
        runs.append(online.run_episode(gm, prior, true_state, K=100, steps=6, config=cfg, seed=5))
        gm.close()
    a, b = runs
    assert a["actions"] == b["actions"] and a["rewards"] == b["rewards"] and a["obs"] == b["obs"]
    assert a["discounted_return"] == b["discounted_return"]
    assert 1 <= a["steps"] <= 6 and all(0 <= x < 13 for x in a["actions"])
    assert all(n > 0 for n in a["survivors"]) or a["deprived"] > 0
