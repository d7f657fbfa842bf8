"""Build an A/B variant of libdespot.so with extra nvcc defines, e.g.
  python scripts/build_variant.py /tmp/libdespot_minb3.so -DHD_CART_MINB=3
then run bench.py with DESPOT_LIB=<path> (despot.py loads that library)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1802_06215_b200 import build as B  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
cmd = [os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *B.NVCC_FLAGS, *extra, "-o", out,
       *[os.path.join(B.CSRC, s) for s in B.SOURCES]]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.stderr.write(res.stderr)
    sys.exit(1)
print(out)
