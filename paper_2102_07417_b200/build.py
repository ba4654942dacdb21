"""Build the in-tree CUDA library (sm_100a) and the oracle's C checker.

``python -m paper_2102_07417_b200.build`` or ``__graft_entry__.build()``.
nvcc cross-compiles without a GPU; the library links the CUDA runtime
statically so the GPU box needs only the driver.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libamgb200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("capi.cu",)]
HEADERS = [os.path.join(CSRC, f) for f in ("kernels.cuh", "halo.h", "setup.cuh")] + [os.path.join(ROOT, "include", "amgb200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
    "-diag-suppress", "550",
]
FSAI_SRC = os.path.join(CSRC, "fsai_host.c")
FSAI_LIB = os.path.join(PKG, "libamgfsai.so")
ORACLE_SRC = os.path.join(ROOT, "oracle", "rowsum.c")
ORACLE_LIB = os.path.join(ROOT, "oracle", "build", "liboracle_rowsum.so")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_library(force=False, verbose=False):
    if force or _stale(LIB, SOURCES + HEADERS):
        cmd = [NVCC] + NVCC_FLAGS + SOURCES + ["-o", LIB]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


CHECKED_LIB = os.path.join(PKG, "libamgb200_checks.so")


def build_checked_library(force=False, verbose=False):
    """libamgb200_checks.so: the same library with device-side invariant checks
    (AMG_CHECK in csrc/kernels.cuh; load it with AMGB200_LIB=... for a test run)."""
    if force or _stale(CHECKED_LIB, SOURCES + HEADERS):
        cmd = [NVCC] + NVCC_FLAGS + ["-DAMG_CHECKS"] + SOURCES + ["-o", CHECKED_LIB]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return CHECKED_LIB


def build_fsai_host(force=False, verbose=False):
    """Host C helper that replays FSAI coefficients when a lean hierarchy cache is loaded."""
    if force or _stale(FSAI_LIB, [FSAI_SRC]):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", FSAI_SRC, "-o", FSAI_LIB, "-lm"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return FSAI_LIB


def build_oracle(force=False):
    """Compile oracle/rowsum.c (the plain-C checker, test infrastructure only)."""
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    if force or _stale(ORACLE_LIB, [ORACLE_SRC]):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", ORACLE_SRC, "-o", ORACLE_LIB],
                       check=True)
    return ORACLE_LIB


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose=True)
    build_fsai_host(force="--force" in sys.argv, verbose=True)
    build_oracle(force="--force" in sys.argv)
    print(LIB)
