"""Scenario sharding across GPUs.

Every rank loads the same belief with despot_opts{rank, world}; the library
keeps the scenarios with global id % world == rank.  A batch then runs
begin (update + expansion + roll-outs + grouping on the local shard) ->
exchange (all-reduce SUM of the exact int64 fixed-point partials and MIN of
the first-occurrence ids, here via torch.distributed / NCCL over NVLink) ->
end (child order, CSR and outputs, identical on every rank).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


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
    sums = torch.as_tensor(_CudaArray(ex.sums, ex.n_sums, "<i8"), device=device)
    mins = torch.as_tensor(_CudaArray(ex.mins, ex.n_mins, "<i4"), device=device)
    return sums, mins


def exchange(sums: torch.Tensor, mins: torch.Tensor, group=None):
    """The one collective step of a sharded batch: exact, order-independent."""
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)


def expand_sharded(model, leaves, group=None, device_outputs=False, child_capacity=None, stream=None):
    batch, ex = model.expand_begin(leaves, stream=stream)
    try:
        sums, mins = exchange_views(ex, torch.device("cuda", model.device))
        exchange(sums, mins, group)
    except Exception:
        model.batch_abort(batch)
        raise
    return model.expand_end(batch, leaves, device_outputs=device_outputs, child_capacity=child_capacity,
                            stream=stream)
