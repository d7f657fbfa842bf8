"""The sharded path end to end with two real processes on one GPU: each rank
loads its scenario shard (despot_opts rank/world), runs begin -> every
exchange round through dist.run_exchange (gloo, device views staged through
host memory; the ranks meet only in host-side collectives) -> end, and gets
the world == 1 result bit for bit -- dense keys (MARS) and the driving
model's sparse keys (record all-gather + merge)."""
import os
import socket

import numpy as np
import pytest
from parity import compare_batch

pytestmark = pytest.mark.gpu

KEYS = ("n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin", "child_count", "child_first",
        "child_weight", "child_upper", "child_lower", "child_obs")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batches():
    from paper_1802_06215_b200 import inputs
    out = []
    kind, params, st, w, seed, _ = inputs.config_inputs(2, K=240, L=8)
    out.append(("mars", kind, params, [(st, w, seed)], "depth1"))
    out.append(("car", "car", inputs.car_params(6, D=25), inputs.car_roots(5, 60, peds=6), "roots"))
    return out


def _run(model, beliefs, mode, sharded, group=None):
    from paper_1802_06215_b200 import inputs
    from paper_1802_06215_b200.dist import expand_sharded
    roots = [model.belief_load(s, w, sd) for s, w, sd in beliefs]
    go = (lambda lv: expand_sharded(model, lv, group, child_capacity=20000)) if sharded else model.expand
    if mode == "roots":
        return [go([(r, -1, 0, 0) for r in roots])]
    R = go([(roots[0], -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], model.A, 8)
    return [R, go([(roots[0], a, c, 1) for a, c in lv])]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1802_06215_b200.despot import Model
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for name, kind, params, beliefs, mode in _batches():
        m = Model(kind, params, rank=rank, world=world)
        res[name] = [{k: np.asarray(o[k]).copy() for k in KEYS} for o in _run(m, beliefs, mode, True)]
        m.close()
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_equal_single_gpu():
    import torch.multiprocessing as mp
    from paper_1802_06215_b200.despot import Model
    ref = {}
    for name, kind, params, beliefs, mode in _batches():
        m = Model(kind, params)
        ref[name] = [{k: np.asarray(o[k]).copy() for k in KEYS} for o in _run(m, beliefs, mode, False)]
        m.close()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    orc = _oracle_results()
    for rank, res in got:
        for name in ref:
            for g, r in zip(res[name], ref[name]):
                for k in KEYS:
                    assert np.array_equal(g[k], r[k]), (rank, name, k)
            for g, (O, om, A) in zip(res[name], orc[name]):  # and against the oracle directly
                compare_batch(g, O, _AOnly(A), om, [(i, i) for i in range(len(O["n_scen"]))])


class _AOnly:
    def __init__(self, A):
        self.A = A


def _oracle_results():
    """The same batches expanded by the CPU oracle (record=True)."""
    import oracle
    from paper_1802_06215_b200 import inputs
    out = {}
    for name, kind, params, beliefs, mode in _batches():
        om = oracle.Model(kind, params)
        roots = [om.belief_load(s, w, sd) for s, w, sd in beliefs]
        if mode == "roots":
            out[name] = [(om.expand([(r, -1, 0, 0) for r in roots], record=True), om, om.A)]
            continue
        R = om.expand([(roots[0], -1, 0, 0)], record=True)
        lv = inputs.select_leaves(R["child_count"], R["child_begin"], om.A, 8)
        out[name] = [(R, om, om.A), (om.expand([(roots[0], a, c, 1) for a, c in lv], record=True), om, om.A)]
    return out
