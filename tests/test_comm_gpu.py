"""The library-owned exchange (despot_opts.comm) on the GPU:
an NCCL communicator created by libdespot (world 1 here -- the pool has one
GPU per call), models loaded with DESPOT_MF_EXCHANGE so that every batch runs
the sharded data path inside despot_expand_batch: dense keys pack the union
of used slots (round A, all-reduce of the flags), all-reduce the packed exact
sums and first ids (round B) and unpack; sparse keys all-gather the record
blocks and merge.  The outputs equal the plain single-GPU path bit for bit
and the CPU oracle within the parity bar; the capacity retry (dense fallback
after an overflowing union) gives the same bits."""
import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import inputs
from paper_1802_06215_b200.despot import DESPOT_MF_EXCHANGE, Comm, Model, comm_unique_id

from parity import compare_batch

pytestmark = pytest.mark.gpu

KEYS = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count", "child_first",
        "child_weight", "child_upper", "child_lower", "child_obs")


@pytest.fixture(scope="module")
def comm():
    import torch.distributed  # noqa: F401  (torch's libnccl in the process)
    c = Comm(comm_unique_id(), 0, 1, 0)
    yield c
    c.close()


def _same(a, b, tag):
    for k in KEYS:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (tag, k)
    assert a["scenario_steps"] == b["scenario_steps"], tag


def _dense_case(comm, cfg, K, L, extra="", D=None):
    kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=K, L=L, D=D)
    plain = Model(kind, params)
    xm = Model(kind, (params + " " + extra).strip(), flags=DESPOT_MF_EXCHANGE, comm=comm)
    om = oracle.Model(kind, params)
    rp, rx, ro = plain.belief_load(st, w, seed), xm.belief_load(st, w, seed), om.belief_load(st, w, seed)
    P0 = plain.expand([(rp, -1, 0, 0)])
    X0 = xm.expand([(rx, -1, 0, 0)], timing=True)
    O0 = om.expand([(ro, -1, 0, 0)], record=True)
    _same(X0, P0, "root")
    compare_batch(X0, O0, xm, om, [(0, 0)])
    assert X0["exchange_rounds"] in (2, 3) and X0["exchange_bytes"] > 0 and X0["exchange_ms"] > 0.0
    lv = inputs.select_leaves(P0["child_count"], P0["child_begin"], plain.A, L)
    P1 = plain.expand([(rp, a, c, 1) for a, c in lv])
    X1 = xm.expand([(rx, a, c, 1) for a, c in lv], timing=True)
    O1 = om.expand([(ro, a, c, 1) for a, c in lv], record=True)
    _same(X1, P1, "depth 1")
    compare_batch(X1, O1, xm, om, [(i, i) for i in range(L)])
    # the dense block the exchange would move vs the packed payload it moved
    LA = L * plain.A
    dense_bytes = 8 * (4 * LA * plain.slots + 3 * LA + 1) + 4 * LA * plain.slots
    return X0, X1, dense_bytes, xm, rx, lv


def test_packed_exchange_mars_equals_single_gpu_and_oracle(comm):
    X0, X1, dense, xm, rx, lv = _dense_case(comm, 2, 200, 16)
    assert X1["exchange_rounds"] == 2  # the capacity hint covers the union
    assert X1["exchange_bytes"] < dense / 2  # compacted: most of the 10 slots per (leaf, action) are empty


def test_packed_exchange_capacity_retry_gives_the_same_bits(comm):
    """xratio16=1: the packed capacity (1/16 slot per (leaf, action) + 256)
    overflows -> every rank falls back to the dense block after the status
    read-back, K3 runs again; the hint then grows so the next batch packs."""
    X0, X1, dense, xm, rx, lv = _dense_case(comm, 3, 150, 12, extra="xratio16=1", D=40)
    assert X0["exchange_rounds"] == 3  # A, B, and the dense fallback
    X2 = xm.expand([(rx, a, c, 1) for a, c in lv])
    assert X2["exchange_rounds"] == 2
    _same(X2, X1, "after the retry")


def test_sparse_exchange_car_equals_single_gpu_and_oracle(comm):
    params = inputs.car_params(6, D=30)
    croots = inputs.car_roots(5, 70, peds=6)
    plain, xm, om = Model("car", params), Model("car", params, flags=DESPOT_MF_EXCHANGE, comm=comm), \
        oracle.Model("car", params)
    rp = [plain.belief_load(s, w_, sd) for s, w_, sd in croots]
    rx = [xm.belief_load(s, w_, sd) for s, w_, sd in croots]
    ro = [om.belief_load(s, w_, sd) for s, w_, sd in croots]
    P0 = plain.expand([(r, -1, 0, 0) for r in rp])
    X0 = xm.expand([(r, -1, 0, 0) for r in rx], timing=True)
    O0 = om.expand([(r, -1, 0, 0) for r in ro], record=True)
    _same(X0, P0, "roots")
    compare_batch(X0, O0, xm, om, [(i, i) for i in range(len(croots))])
    assert X0["exchange_rounds"] == 1 and X0["exchange_bytes"] > 0
    R = plain.expand([(rp[0], -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], plain.A, 6)
    xm.expand([(rx[0], -1, 0, 0)])
    om.expand([(ro[0], -1, 0, 0)])
    P1 = plain.expand([(rp[0], a, c, 1) for a, c in lv])
    X1 = xm.expand([(rx[0], a, c, 1) for a, c in lv])
    O1 = om.expand([(ro[0], a, c, 1) for a, c in lv], record=True)
    _same(X1, P1, "children")
    compare_batch(X1, O1, xm, om, [(i, i) for i in range(len(lv))])


def test_rollout_bounds_through_the_communicator(comm):
    kind, params, st, w, seed, _ = inputs.config_inputs(1, K=90)
    plain, xm = Model(kind, params), Model(kind, params, flags=DESPOT_MF_EXCHANGE, comm=comm)
    a = plain.rollout_bounds(plain.belief_load(st, w, seed))
    b = xm.rollout_bounds(xm.belief_load(st, w, seed))
    assert a == b


def test_comm_info_and_model_mismatch(comm):
    info = comm.info()
    assert info["rank"] == 0 and info["world"] == 1 and info["nccl_version"] >= 22000
    from paper_1802_06215_b200.despot import DespotError
    with pytest.raises(DespotError):
        Model("tiger", inputs.tiger_params(), rank=0, world=2, comm=comm)  # the comm has 1 rank
