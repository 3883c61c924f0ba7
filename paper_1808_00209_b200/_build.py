"""Builds libbnn.so in-tree with nvcc for sm_100a (B200) only.

    python -m paper_1808_00209_b200._build [--force]

No PTX / other-arch fallback: `-gencode arch=compute_100a,code=sm_100a`.  The CUDA runtime is
linked statically so the library does not depend on which libcudart the host process loaded.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libbnn.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(INCLUDE, "bnn.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


TRACE_LIB = os.path.join(PKG, "libbnn_trace.so")  # diagnostics build (-DBNN_TRACE: bnn_set_trace records)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    out = TRACE_LIB if trace else LIB
    if not trace and not force and not needs_build():
        return LIB
    tmp = out + ".tmp%d" % os.getpid()
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-DBNN_TRACE=1"] if trace else []), "-I", INCLUDE, "-I", CSRC, "-o", tmp,
           os.path.join(CSRC, "bnn_api.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
