"""The N>1 exchange step with the gloo backend, world size 2,
on CPU: every rank contributes exact int64 fixed-point partials and int32
first-occurrence ids; after `dist.exchange` every rank holds the elementwise
sum / min, identical on all ranks and independent of the reduction order."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_06215_b200 import dist as ddist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partials(rank, n_sums=1000, n_mins=300):
    rng = np.random.default_rng(100 + rank)
    sums = rng.integers(-2**58, 2**58, n_sums, dtype=np.int64)
    mins = rng.integers(0, 2**31 - 1, n_mins, dtype=np.int64).astype(np.int32)
    mins[rng.random(n_mins) < 0.3] = 0x7F7F7F7F  # empty slots on this shard (memset sentinel)
    return sums, mins


def _block(rank, nbytes=1024):
    """this rank's all-gather block (the sparse-key records, §6.2)"""
    return np.random.default_rng(500 + rank).integers(0, 256, nbytes, dtype=np.uint8)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, m = _partials(rank)
    ts, tm = torch.from_numpy(s.copy()), torch.from_numpy(m.copy())
    ddist.exchange(ts, tm)
    # the sparse-key rounds: MAX of (record count, largest child set), then
    # the in-place all-gather of every rank's block
    tx = torch.tensor([100 + 7 * rank, 3 - rank], dtype=torch.int64)
    blk = _block(rank)
    g = torch.zeros(world * blk.size, dtype=torch.uint8)
    g[rank * blk.size:(rank + 1) * blk.size] = torch.from_numpy(blk)
    ddist.exchange(None, None, maxs=tx, gather=g)
    q.put((rank, ts.numpy().copy(), tm.numpy().copy(), tx.numpy().copy(), g.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_sum_min_max_gather_world2_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = [_partials(r) for r in range(world)]
    want_s = sum(p[0] for p in parts)  # int64 wrap-around arithmetic is exact either way
    want_m = np.minimum(parts[0][1], parts[1][1])
    want_x = np.array([100 + 7 * (world - 1), 3], dtype=np.int64)
    want_g = np.concatenate([_block(r) for r in range(world)])
    for _, s, m, x, g in res:
        assert np.array_equal(s, want_s)
        assert np.array_equal(m, want_m)
        assert np.array_equal(x, want_x)
        assert np.array_equal(g, want_g)
    # order independence: reversing the ranks' contributions gives the same bits
    assert np.array_equal(parts[1][0] + parts[0][0], want_s)


def test_shard_rule_partitions_ids():
    """global id % world == rank: every id on exactly one rank, ascending per rank"""
    K = 1037
    for world in (1, 2, 3, 8):
        seen = np.concatenate([ddist.shard_ids(K, r, world) for r in range(world)])
        assert np.array_equal(np.sort(seen), np.arange(K))
        for r in range(world):
            ids = ddist.shard_ids(K, r, world)
            assert np.all(np.diff(ids) > 0) and np.all(ids % world == r)


def _boot_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = ddist.bootstrap_unique_id()
    q.put((rank, uid))
    dist.barrier()
    dist.destroy_process_group()


def test_communicator_bootstrap_world2_gloo():
    """SURVEY §8(e) bootstrap of the library's NCCL communicator: rank 0's
    ncclGetUniqueId (through libdespot, NCCL resolved at run time) reaches
    every rank over the process group, byte for byte.  (ncclCommInitRank
    itself needs the GPUs.)"""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_boot_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1] and any(got[0])
