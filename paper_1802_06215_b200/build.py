"""Build libdespot.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdespot.so")
SOURCES = ["despot.cu", "search.cpp"]
def _nccl_include():
    """nccl.h for the types (NCCL itself is loaded at run time, nccl_dl.h):
    the torch-bundled NCCL's headers, else the system's."""
    try:
        import nvidia.nccl
        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit-exact fp32 model arithmetic (R16): no FMA contraction,
    # IEEE division / square root, no flush-to-zero
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-cudart", "static", "-shared",
    "-Xptxas", "-v",
    "-I" + _nccl_include(), "-ldl",
]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "despot.h"))
    files.append(os.path.abspath(__file__))
    return files


CHECKED = os.path.join(HERE, "libdespot_checked.so")


def build_checked(force: bool = False) -> str:
    """The self-check build (-DHD_CHECKS: device checks of index and protocol
    invariants; common.cuh), loaded by the self-check tests through DESPOT_LIB."""
    if not force and os.path.exists(CHECKED) and all(os.path.getmtime(CHECKED) >= os.path.getmtime(f) for f in _deps()):
        return CHECKED
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = CHECKED + f".tmp{os.getpid()}"
    cmd = [nvcc, *[f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-DHD_CHECKS", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libdespot_checked.so")
    os.replace(tmp, CHECKED)
    return CHECKED


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(f) for f in _deps()):
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libdespot.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:  # registers / spills / smem per kernel
        f.write("".join(l for l in res.stderr.splitlines(True) if "Compile time" not in l))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
