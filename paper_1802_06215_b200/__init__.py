"""B200-native batched leaf expansion of HyP-DESPOT (arXiv 1802.06215).

The product is libdespot.so (C ABI in include/despot.h, sm_100a kernels in
csrc/); `despot` is its thin ctypes binding, `dist` the scenario-sharded
multi-GPU exchange, `inputs` the seeded synthetic workloads.
"""
from .despot import DespotError, Model  # noqa: F401

__all__ = ["Model", "DespotError"]
