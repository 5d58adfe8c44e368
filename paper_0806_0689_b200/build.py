"""Build libme.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and the tests."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libme.so")
SO_DEBUG = os.path.join(HERE, "libme_debug.so")  # -DME_DEBUG: device bounds checks
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "me.h")])


def stale(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(f) > t for f in sources())


def build(force: bool = False, verbose: bool = False, extra=(), debug: bool = False) -> str:
    """libme.so, or with debug=True libme_debug.so (ME_DEBUG bounds checks in the kernels)."""
    so = SO_DEBUG if debug else SO
    if not force and not stale(so):
        return so
    tmp = so + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, *(["-DME_DEBUG"] if debug else []), *extra, "-o", tmp,
           os.path.join(CSRC, "me_api.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv,
                extra=["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else []))
