"""GPU parity (-m gpu) of the header-only device API include/squares_dev.cuh:
sq::squares32 / sq::squares64 on explicit pairs and sq::Stream (next_u32/u64/f32/f64, skip)
inside a user kernel, bit-exact against the oracle."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
import synth_inputs as SI

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def lib():
    from paper_2004_06278_b200 import _build
    path = _build.build_devapi_test()
    L = ctypes.CDLL(path)
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    L.devapi_pairs.argtypes = [vp, vp, u64, vp, vp]
    L.devapi_stream.argtypes = [u64, u64, u64, u64, ctypes.c_int, u64, vp]
    torch.cuda.set_device(0)
    return L


def test_pairs(lib):
    ctr, key = SI.random_pairs(200_000, seed=77)
    c = torch.from_numpy(ctr.view(np.int64)).cuda()
    k = torch.from_numpy(key.view(np.int64)).cuda()
    o32 = torch.empty(ctr.size, dtype=torch.int32, device="cuda")
    o64 = torch.empty(ctr.size, dtype=torch.int64, device="cuda")
    assert lib.devapi_pairs(c.data_ptr(), k.data_ptr(), ctr.size, o32.data_ptr(), o64.data_ptr()) == 0
    assert np.array_equal(o32.cpu().numpy().view(np.uint32), O.squares_pairs(ctr, key, 32))
    assert np.array_equal(o64.cpu().numpy().view(np.uint64), O.squares_pairs(ctr, key, 64))


@pytest.mark.parametrize("kind,dt", [(0, torch.int32), (1, torch.int64), (2, torch.float32), (3, torch.float64)])
@pytest.mark.parametrize("skip0", [0, 5, 1 << 40])
def test_stream(lib, kind, dt, skip0):
    key = int(O.keygen(3, 1)[0])
    ctr0, per, threads = M64 - 5000, 37, 1000
    out = torch.empty(per * threads, dtype=dt, device="cuda")
    assert lib.devapi_stream(key, ctr0, per, skip0, kind, threads, out.data_ptr()) == 0
    got = out.cpu().numpy()
    name = ["u32", "u64", "f32", "f64"][kind]
    for t in (0, 1, 499, threads - 1):
        want = O.fill(name, [key], ctr0 + t * per + skip0, per)[0]
        assert np.array_equal(got[t * per:(t + 1) * per].view(np.uint8), want.view(np.uint8)), (t, skip0)
