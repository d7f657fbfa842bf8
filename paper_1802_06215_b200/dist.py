"""Scenario sharding across GPUs.

Every rank loads the same belief with despot_opts{rank, world}; the library
keeps the scenarios with global id % world == rank.

The primary form is library-owned: `init_comm` bootstraps an NCCL
communicator inside libdespot (rank 0's unique id broadcast over the torch
process group), models are loaded with it, and `Model.expand` runs the whole
sharded batch -- update, expansion, roll-outs, grouping, the exchange on the
batch's stream (dense keys: all-reduce of the union of used slots, then of
the packed exact int64 sums and first ids; sparse keys: SUM of the per-action
partials and an all-gather of the ranks' child records), finalize -- in one
call, with no Python between K2 and K3.

The caller-driven form (begin -> `run_exchange` -> end) remains for a
transport of the caller's choosing, e.g. gloo with host-staged device views
(the CPU and two-process tests): one round of in-place collectives.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def bootstrap_unique_id(group=None) -> bytes:
    """Rank 0's 128-byte NCCL unique id on every rank (broadcast over the
    process group; gloo or nccl)."""
    from .despot import comm_unique_id
    rank = dist.get_rank(group)
    src = dist.get_global_rank(group, 0) if group is not None else 0
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(comm_unique_id()), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        t = uid.cuda()
        dist.broadcast(t, src=src, group=group)
        uid = t.cpu()
    else:
        dist.broadcast(uid, src=src, group=group)
    return bytes(uid.numpy().tobytes())


def init_comm(group=None, device: int = 0):
    """The library's communicator for this rank (SURVEY §8(e) bootstrap:
    torch process group -> ncclGetUniqueId on rank 0 -> broadcast ->
    ncclCommInitRank inside libdespot)."""
    from .despot import Comm
    uid = bootstrap_unique_id(group)
    return Comm(uid, dist.get_rank(group), dist.get_world_size(group), device)


def shard_ids(K: int, rank: int, world: int):
    """Global scenario ids kept by `rank` (the rule despot_belief_load applies)."""
    import numpy as np
    return np.arange(rank, K, world, dtype=np.int64)


class _CudaArray:
    """Zero-copy view of a device buffer owned by libdespot."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def exchange_views(ex, device):
    """(sums, mins) views of a dense-key exchange round (kept for callers of
    the one-round form); see round_views for every collective of a round."""
    v = round_views(ex, device)
    return v["sums"], v["mins"]


def round_views(ex, device):
    """Zero-copy tensors of one exchange round: sums (SUM), mins (MIN), maxs
    (MAX), gather (all-gather, uint8 [world * gather_bytes]); None if unused."""
    def view(ptr, n, typestr):
        return torch.as_tensor(_CudaArray(ptr, n, typestr), device=device) if ptr and n else None
    return {"sums": view(ex.sums, ex.n_sums, "<i8"), "mins": view(ex.mins, ex.n_mins, "<i4"),
            "maxs": view(ex.maxs, ex.n_maxs, "<i8"), "gather": None if not ex.gather_bytes else
            (int(ex.gather), int(ex.gather_bytes))}


def exchange(sums: torch.Tensor, mins: torch.Tensor, group=None, maxs=None, gather=None):
    """The collectives of one exchange round, in place: exact integer sums and
    minima (order-independent; `maxs` only for ABI-1 callers), and the
    all-gather of the ranks' blocks (`gather` = the whole [world * block] byte tensor; this rank's block
    is already filled).  NCCL works on the device views directly; a host
    backend (gloo: the CPU tests, or device tensors staged through host
    memory) gets host copies."""
    nccl = dist.get_backend(group) == "nccl"

    def reduce(t, op):
        if t is None:
            return
        if nccl or not t.is_cuda:
            dist.all_reduce(t, op=op, group=group)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=group)
            t.copy_(h)

    reduce(sums, dist.ReduceOp.SUM)
    reduce(mins, dist.ReduceOp.MIN)
    reduce(maxs, dist.ReduceOp.MAX)
    if gather is not None:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        blk = gather.numel() // world
        if nccl:
            dist.all_gather_into_tensor(gather, gather[rank * blk:(rank + 1) * blk].clone(), group=group)
        else:  # list form on host memory
            h = gather.cpu() if gather.is_cuda else gather
            parts = list(h.split(blk))
            dist.all_gather(parts, h[rank * blk:(rank + 1) * blk].clone(), group=group)
            if gather.is_cuda:
                gather.copy_(h)


def run_exchange(model, batch, ex, group=None):
    """The exchange round(s) of a caller-driven sharded batch (one in ABI 2)."""
    device = torch.device("cuda", model.device)
    world = dist.get_world_size(group)
    while True:
        v = round_views(ex, device)
        gather = None
        if v["gather"] is not None:
            ptr, blk = v["gather"]
            gather = torch.as_tensor(_CudaArray(ptr, world * blk, "|u1"), device=device)
        exchange(v["sums"], v["mins"], group, maxs=v["maxs"], gather=gather)
        if not ex.more:
            return
        ex = model.batch_exchange(batch)


def _torch_stream(stream, device):
    """The torch stream object of the batch's stream (None: torch's current
    stream, which is also what the binding hands the library)."""
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(getattr(stream, "cuda_stream", stream)), device=device)


def expand_sharded(model, leaves, group=None, device_outputs=False, child_capacity=None, stream=None):
    if model.comm is not None:  # library-owned exchange: one call
        return model.expand(leaves, device_outputs=device_outputs, child_capacity=child_capacity, stream=stream)
    batch, ex = model.expand_begin(leaves, stream=stream)
    try:
        # the collectives run on the batch's own stream (ordered after K2 and
        # before K3; a host backend's staging copies synchronise that stream)
        with torch.cuda.stream(_torch_stream(stream, torch.device("cuda", model.device))):
            run_exchange(model, batch, ex, group)
    except Exception:
        model.batch_abort(batch)
        raise
    return model.expand_end(batch, leaves, device_outputs=device_outputs, child_capacity=child_capacity,
                            stream=stream)
