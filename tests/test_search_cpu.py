"""The host tree driver (despot_search, include/despot.h) on CPU, with the
oracle plugged in as the expansion backend (test infrastructure only; the
product backend is libdespot's GPU expansion, tests/test_search_gpu.py).

Checks: convergence of the anytime search to the brute-force optimal value of
the D-truncated DESPOT (Eq. 4 backups of valid bounds), the bound
invariant l <= V* <= u, count consistency sum_a N(b,a) = N(b) and released
virtual-loss markers after multi-worker runs, determinism of the
serial search, and the root action argmax_a l(b0, a)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import build as B
from paper_1802_06215_b200 import despot as D
from paper_1802_06215_b200 import inputs


@pytest.fixture(scope="module", autouse=True)
def _built():
    B.build()


class OracleBackend:
    """despot_expand_fn / despot_release_fn backed by oracle.Model."""

    def __init__(self, om: oracle.Model):
        import threading
        self.om = om
        self.lock = threading.Lock()  # the oracle is single-threaded; the search may call from two batchers
        self.calls = 0
        self.leaves_seen = 0
        self.released = []
        self._expand = D.EXPAND_FN(self.expand)
        self._release = D.RELEASE_FN(self.release)

    def expand(self, ctx, leaves_p, L, out_p):
        with self.lock:
            return self._expand_locked(ctx, leaves_p, L, out_p)

    def _expand_locked(self, ctx, leaves_p, L, out_p):
        try:
            lv = C.cast(leaves_p, C.POINTER(D.Leaf))
            out = C.cast(out_p, C.POINTER(D.Expansion)).contents
            leaves = [(lv[i].parent, lv[i].action, lv[i].child, lv[i].depth) for i in range(L)]
            o = self.om.expand(leaves, child_capacity=out.child_capacity)
            A, OW = self.om.A, self.om.OW
            nc = int(o["child_begin"][-1])

            def put(ptr, arr, ctype):
                if len(arr):
                    np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (len(arr),))[:] = arr

            put(out.node, np.asarray(o["node"], np.uint64), C.c_uint64)
            put(out.n_scen, o["n_scen"], C.c_uint32)
            put(out.weight, o["weight"].astype(np.float32), C.c_float)
            put(out.act_reward, o["act_reward"].astype(np.float32), C.c_float)
            put(out.act_upper, o["act_upper"].astype(np.float32), C.c_float)
            put(out.act_lower, o["act_lower"].astype(np.float32), C.c_float)
            put(out.child_begin, o["child_begin"], C.c_uint32)
            put(out.child_count, o["child_count"][:nc], C.c_uint32)
            put(out.child_first, o["child_first"][:nc], C.c_uint32)
            put(out.child_weight, o["child_weight"][:nc].astype(np.float32), C.c_float)
            put(out.child_upper, o["child_upper"][:nc].astype(np.float32), C.c_float)
            put(out.child_lower, o["child_lower"][:nc].astype(np.float32), C.c_float)
            put(out.child_obs, o["child_obs"][:nc].reshape(-1), C.c_uint32)
            out.scenario_steps = o["scenario_steps"]
            out.num_children = nc
            self.calls += 1
            self.leaves_seen += L
            assert len(o["node"]) == L and A and OW
            return 0
        except Exception as e:  # never raise through the C frame
            print("backend error", e)
            return -1

    def release(self, ctx, node):
        self.released.append(int(node))
        return 0

    def problem(self, root, root_upper, root_lower, depth=0, K=1):
        om = self.om
        return D.SearchProblem(om.A, om.OW, om.slots, om.D, om.gamma, root, depth, K, 0.0, root_upper, root_lower,
                               C.cast(self._expand, C.c_void_p), C.cast(self._release, C.c_void_p), None)


def run(kind, params, st, w, seed, cfg, dump=100000):
    om = oracle.Model(kind, params)
    root = om.belief_load(st, w, seed)
    u0, l0 = om.rollout_bounds(root)
    be = OracleBackend(om)
    res, nodes = D.search(be.problem(root, u0, l0, K=len(w)), cfg, dump_capacity=dump)
    return om, root, be, res, nodes


def check_invariants(nodes, tol=1e-5):
    n = [x for x in nodes if x.depth or x.parent == -1]
    for x in n:
        assert x.active == 0, "virtual-loss markers must all be released"
        if x.expanded:
            assert x.visits == x.branch_visits, "sum_a N(b,a) = N(b)"
        assert x.lower <= x.upper + tol * max(1.0, abs(x.upper))
        assert x.lower >= x.lower0 - tol * max(1.0, abs(x.lower0))  # floored at the initial bound
        assert x.upper <= x.upper0 + tol * max(1.0, abs(x.upper0))  # capped by the initial bound


def test_serial_search_converges_to_brute_force_tiger():
    st = np.array([[0, 1, 1, 0, 1, 1, 0, 1]], np.uint32)
    w = inputs.weights(8)
    cfg = D.search_config(workers=1, max_inflight=1, max_batch=1, max_trials=2000, xi=0.5)
    om, root, be, res, nodes = run("tiger", inputs.tiger_params(D=4), st, w, 5, cfg)
    v = om.brute_force(root)
    q = om.brute_force_q(root)
    assert abs(res["root_lower"] - v) < 1e-4 and abs(res["root_upper"] - v) < 1e-4, (res, v)
    assert res["action"] == int(np.argmax(q))
    assert res["nodes"] == len(nodes)
    check_invariants(nodes)
    # every node the search created on the backend is released (not the root)
    assert sorted(be.released) == sorted(set(be.released)) and root not in be.released
    assert len(be.released) == res["expanded"] - 1


@pytest.mark.parametrize("case", ["rocksample", "nav", "car"])
def test_parallel_search_bounds_and_counts(case):
    if case == "rocksample":
        kind, params = "rocksample", "n=3 robots=1 D=4 gamma=0.95 rocks=1:0,2:2 starts=0:1"
        st = np.zeros((2, 6), np.uint32)
        st[0] = [0, 1, 2, 3, 1, 2]
        st[1] = 3
    elif case == "nav":
        kind, params = "nav", inputs.nav_params(5, wall_y=2, gates=(1, 3), landmarks=[], goal=(2, 4), D=4)
        rng = np.random.default_rng(2)
        st = np.zeros((2, 5), np.uint32)
        st[0] = rng.integers(0, 5, 5) + (rng.integers(0, 2, 5) << 8)
        st[1] = (rng.random((5, 10)) < 0.1).astype(np.uint32) @ (1 << np.arange(10, dtype=np.uint32))
    else:
        kind, params = "car", inputs.car_params(peds=2, D=4)
        st = inputs.car_belief(5, 3, peds=2)
        st[0] = np.float32(18.75).view(np.uint32)
        st[1] = 3
    K = st.shape[1]
    w = inputs.weights(K, 9, uniform=False)
    cfg = D.search_config(workers=4, max_inflight=4, max_batch=8, batch_wait_us=100, max_trials=600, xi=0.3,
                          c_a=0.5, c_o=0.2)
    om, root, be, res, nodes = run(kind, params, st, w, 11, cfg)
    check_invariants(nodes)
    v = om.brute_force(root)
    tol = 1e-5 * max(1.0, abs(v))  # the backend's outputs are fp32 (R12)
    assert res["root_lower"] <= v + tol and v <= res["root_upper"] + tol, (res, v)
    assert res["batches"] == be.calls and res["expanded"] == be.leaves_seen
    # the trial budget is spent, or the search stopped early on a closed root gap
    assert res["trials"] == 600 or res["root_upper"] - res["root_lower"] <= tol, res


def test_serial_search_is_deterministic():
    kind, params, st, w, seed, _ = inputs.config_inputs(1, K=30, D=8)
    cfg = D.search_config(workers=1, max_inflight=1, max_batch=1, max_trials=150, xi=0.9, c_a=1.0)
    a = run(kind, params, st, w, seed, cfg)
    b = run(kind, params, st, w, seed, cfg)
    assert a[3]["nodes"] == b[3]["nodes"] and a[3]["action"] == b[3]["action"]
    fa = [(x.parent, x.action, x.child, x.visits, x.upper, x.lower) for x in a[4]]
    fb = [(x.parent, x.action, x.child, x.visits, x.upper, x.lower) for x in b[4]]
    assert fa == fb


def test_search_rejects_bad_problems():
    om = oracle.Model("tiger", inputs.tiger_params(D=3))
    be = OracleBackend(om)
    p = be.problem(1, 10.0, -3.0, depth=3)  # root at depth D
    with pytest.raises(D.DespotError):
        D.search(p, D.search_config(max_trials=1))
