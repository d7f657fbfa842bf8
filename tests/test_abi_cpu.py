"""CPU-side checks of the boundary: libdespot.so builds for sm_100a, loads, and
exports every entry point include/despot.h declares; without a GPU it fails
loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_1802_06215_b200 import build as B
from paper_1802_06215_b200 import despot

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "despot.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(despot_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    path = B.build()
    lib = ctypes.CDLL(path)
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/despot.h but not exported"
    assert sorted(despot.EXPORTS) == names
    lib.despot_abi_version.restype = ctypes.c_int
    assert lib.despot_abi_version() == 2


def test_cubin_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(despot.DespotError) as e:
        despot.Model("rocksample", "n=7 robots=1 rocks=2:0 starts=0:3")
    assert e.value.code == -5  # DESPOT_ECUDA


def test_bad_params_rejected_before_device_use():
    with pytest.raises(despot.DespotError) as e:
        despot.Model("no_such_model", "")
    assert e.value.code == -1
    with pytest.raises(despot.DespotError) as e:
        despot.Model("rocksample", "n=7 robots=1 rocks=2:0,2:0 starts=0:3")  # two rocks on one cell
    assert e.value.code == -1


def test_nccl_unique_id_without_a_gpu():
    """despot_comm_unique_id resolves NCCL at run time (the torch-bundled copy
    here) and needs no device: the bootstrap step of the multi-GPU path."""
    import torch.distributed  # noqa: F401  (loads torch's libnccl into the process)
    a, b = despot.comm_unique_id(), despot.comm_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
