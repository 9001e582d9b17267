"""Build libpic.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import glob
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
LIB = os.path.join(_HERE, "libpic.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-diag-suppress", "550",
]


def nccl_dirs():
    """NCCL 2.28 headers and library bundled with torch (nvidia-nccl-cu12 wheel)."""
    import nvidia.nccl as m

    root = os.path.dirname(m.__file__) if getattr(m, "__file__", None) else list(m.__path__)[0]
    return os.path.join(root, "include"), os.path.join(root, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(_HERE, "..", "include", "*.h")))


def build_lib(force: bool = False, verbose: bool = False) -> str:
    srcs = sources()
    if not force and os.path.exists(LIB):
        newest = max(os.path.getmtime(p) for p in srcs + headers())
        if os.path.getmtime(LIB) >= newest:
            return LIB
    inc, libdir = nccl_dirs()
    extra = os.environ.get("PIC_NVCC_EXTRA", "").split()   # tuning experiments, e.g. -DPIC_X=1
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-I" + inc, "-o", LIB, *srcs, "-L" + libdir, "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + libdir]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return LIB
