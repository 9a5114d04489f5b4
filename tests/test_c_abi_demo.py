"""The C ABI used from plain C (examples/c_abi_demo.c): it compiles against include/squares.h and
links libsquares.so with gcc on CPU; on a GPU (-m gpu) its printed outputs equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_06278_b200")


def _build(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    exe = str(tmp_path / "c_abi_demo")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", LIBDIR, "-lsquares",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs_bit_exact(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = dict(ln.split(" ", 1) for ln in r.stdout.strip().splitlines() if " " in ln)
    keys = O.keygen(1, 4)
    assert lines["key"].split()[0] == f"{int(keys[0]):016x}"
    want_u = O.fill("u32", [int(keys[0])], 0, 4)[0]
    assert [int(x, 16) for x in lines["u32"].split()] == [int(x) for x in want_u]
    want_f = O.fill("f32", keys, 0, 4)[1]
    assert np.array_equal(np.array([float(x) for x in lines["f32"].split()], np.float32), want_f)
    assert r.stdout.strip().endswith("ok")
