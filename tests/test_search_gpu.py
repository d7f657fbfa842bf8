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
