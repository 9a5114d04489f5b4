"""Builds libsquares.so in-tree: nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_2004_06278_b200._build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsquares.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["capi.cu", "fill.cu", "fused.cu", "keyctr.cu", "scaled.cu", "keygen.cpp"]
HEADERS = ["sq_internal.h", "hist16.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "squares.h"))
    deps.append(os.path.join(os.path.dirname(PKG), "include", "squares_dev.cuh"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None, extra=()) -> str:
    """Compile libsquares.so (or, for experiments, a variant with extra -D defines at `out`)."""
    lib = out or LIB
    if not force and not defines and not extra and out is None and not _stale():
        return LIB
    tag = "_".join([d.replace("=", "") for d in defines] + [e.strip("-").replace(" ", "") for e in extra]) or "default"
    objdir = os.path.join(PKG, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libsquares.so failed")
    os.replace(tmp, lib)
    return lib


DEVTEST_SRC = os.path.join(os.path.dirname(PKG), "tests", "devapi_kernels.cu")
DEVTEST_LIB = os.path.join(os.path.dirname(PKG), "tests", "libdevapi_test.so")


def build_devapi_test(force: bool = False) -> str:
    """Test kernels that exercise the header-only device API (include/squares_dev.cuh)."""
    hdr = os.path.join(os.path.dirname(PKG), "include", "squares_dev.cuh")
    if (not force and os.path.exists(DEVTEST_LIB)
            and os.path.getmtime(DEVTEST_LIB) > max(os.path.getmtime(DEVTEST_SRC), os.path.getmtime(hdr))):
        return DEVTEST_LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-o", DEVTEST_LIB, DEVTEST_SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed on tests/devapi_kernels.cu")
    return DEVTEST_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
