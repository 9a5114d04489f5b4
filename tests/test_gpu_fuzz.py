"""Seeded randomized parity (-m gpu): 60 fill cases and 24 fused cases drawn over the whole
argument space -- every output kind, device keys or key by value, counter starts anywhere in
[0, 2^64) (wrap included), strides (including huge ones), ragged lengths, row pitches with
padding, misaligned output offsets -- each compared bit-exactly with the oracle.  The draws come
from numpy's PCG64 with the documented parity seed 20040627 (synth_inputs), so a failure is
reproducible from its case index."""
import numpy as np
import pytest
import torch

import oracle as O
import oracle.battery as OB

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1
KINDS = ["u32", "u64", "f32", "f64", "f32x2"]
ES = {"u32": 4, "u64": 8, "f32": 4, "f64": 8, "f32x2": 8}


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    torch.cuda.set_device(0)
    return sq


def _pick(rng, items):
    """One element of a Python list (exact big ints: numpy's choice would go through float64)."""
    return items[int(rng.integers(0, len(items)))]


def _case(i, salt):
    rng = np.random.default_rng([20040627, salt, i])
    ctr0 = int(rng.integers(0, 1 << 63)) * 2 + int(rng.integers(0, 2))
    if rng.random() < 0.25:                       # near the 2^64 wrap
        ctr0 = M64 - int(rng.integers(0, 5000))
    n = _pick(rng, [1, 2, 5, 31, 511, 512, 513, 4097, int(rng.integers(1, 200_000))])
    stride = _pick(rng, [1, 1, 1, 2, 3, 255, 1 << 32, M64, int(rng.integers(1, 1 << 62))])
    return rng, ctr0, n, stride


@pytest.mark.parametrize("i", range(60))
def test_fill_fuzz(sq, i):
    rng, ctr0, n, stride = _case(i, 1)
    kind = KINDS[i % len(KINDS)]
    es = ES[kind]
    by_value = rng.random() < 0.3
    nkeys = 1 if by_value else int(rng.integers(1, 5))
    pad = 0 if nkeys == 1 else int(rng.integers(0, 40))
    ld = n + pad
    off = int(rng.integers(0, 8))                  # elements: misaligned to 32 B for most values
    keys = O.keygen(int(rng.integers(0, 1 << 31)), nkeys)
    if rng.random() < 0.1:
        keys = np.array([0, 1, 1 << 32, M64][:nkeys], dtype=np.uint64) if nkeys <= 4 else keys
    words = es // 4
    buf = torch.full(((off + nkeys * ld) * words + 64,), -1, dtype=torch.int32, device="cuda")
    dt = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32, "f64": torch.float64,
          "f32x2": torch.float32}[kind]
    view = buf[off * words: (off + nkeys * ld) * words].view(dt)
    if kind == "f32x2":
        view = view.view(nkeys, ld, 2)
    else:
        view = view.view(nkeys, ld)
    if by_value:
        sq.fill_ex(kind, ctr0, n, stride=stride, key=int(keys[0]), out=view.reshape(-1) if kind != "f32x2" else view.reshape(-1, 2))
    else:
        kd = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).cuda()
        sq.fill_ex(kind, ctr0, n, stride=stride, keys=kd, out=view, ld=ld)
    torch.cuda.synchronize()
    allw = buf.cpu().numpy().view(np.uint32)
    got = allw[off * words: (off + nkeys * ld) * words].reshape(nkeys, ld * words)
    want = O.fill_strided(kind, keys, ctr0, stride, n)
    want_w = np.ascontiguousarray(want).view(np.uint32).reshape(nkeys, n * words)
    assert np.array_equal(got[:, :n * words], want_w), (i, kind, ctr0, n, stride, nkeys, ld, off)
    assert (got[:, n * words:] == 0xFFFFFFFF).all(), ("padding written", i)
    assert (allw[:off * words] == 0xFFFFFFFF).all() and (allw[(off + nkeys * ld) * words:] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("i", range(24))
def test_fused_fuzz(sq, i):
    rng, ctr0, n, stride = _case(i, 2)
    n = _pick(rng, [1, 33, 4096, int(rng.integers(1, 1 << 21))])
    bitrev = bool(rng.random() < 0.4)
    key = int(O.keygen(int(rng.integers(0, 1 << 31)), 1)[0]) if rng.random() < 0.8 else _pick(rng, [0, 1, 1 << 32])
    h0 = torch.from_numpy(rng.integers(0, 1 << 40, 65536).astype(np.int64)).cuda()   # accumulate onto
    o0 = torch.from_numpy(rng.integers(0, 1 << 40, 32).astype(np.int64)).cuda()      # non-zero arrays
    h, o = h0.clone(), o0.clone()
    sq.fused_stats_ex(key, ctr0, n, stride=stride, bitrev=bitrev, hist=h, ones=o)
    torch.cuda.synchronize()
    hw, ow = O.fused_stats_ex(key, ctr0, stride, n, bitrev)
    assert np.array_equal((h - h0).cpu().numpy().view(np.uint64), hw), (i, ctr0, n, stride, bitrev, key)
    assert np.array_equal((o - o0).cpu().numpy().view(np.uint64), ow), (i, ctr0, n, stride, bitrev, key)


@pytest.mark.parametrize("i", range(16))
def test_transitions_fuzz(sq, i):
    """sq_transitions (runs statistic) on ragged lengths (n < 8, n % 8 != 0: the scalar tail and
    the per-thread boundary pairs), strides, bit reversal, accumulation onto a non-zero count;
    against the oracle stream's direct bit comparison."""
    rng, ctr0, n, stride = _case(i, 3)
    n = _pick(rng, [1, 2, 7, 8, 9, 255, 4103, int(rng.integers(1, 300_000))])
    bitrev = bool(rng.random() < 0.5)
    key = int(O.keygen(int(rng.integers(0, 1 << 31)), 1)[0])
    c = torch.full((1,), 1 << 40, dtype=torch.int64, device="cuda")
    sq.transitions(key, ctr0, n, stride=stride, bitrev=bitrev, count=c)
    torch.cuda.synchronize()
    w = O.fill_strided("u32", [key], ctr0, stride, n)[0]
    if bitrev:
        w = np.array([O.bitrev32(int(x)) for x in w], np.uint32)
    assert int(c.item()) - (1 << 40) == OB.counts(w)["transitions"], (i, ctr0, n, stride, bitrev)
