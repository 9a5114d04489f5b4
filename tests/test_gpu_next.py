"""GPU parity (-m gpu) of the SURVEY 8(f) entry points vs the oracle, bit-exact:
squares64-derived floats (f64, f32x2), strided counters (sq_fill_ex), key-counter mode
(sq_fill_keyctr) and the strided / bits-reversed fused statistics (sq_fused_stats_ex)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth_inputs as SI
from tests.helpers import first_mismatch

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    torch.cuda.set_device(0)
    return sq


def _dev_keys(k):
    return torch.from_numpy(np.ascontiguousarray(k, dtype=np.uint64).view(np.int64)).cuda()


def _raw(t):
    a = t.cpu().numpy()
    return a.view(np.uint64) if a.dtype.itemsize == 8 or a.ndim == 3 else a.view(np.uint32)


@pytest.mark.parametrize("kind", ["f64", "f32x2"])
@pytest.mark.parametrize("ctr0,n,nkeys,pad", [(0, 1 << 20, 1, 0), (M64 - 999, 4099, 3, 5), (7, 1, 1, 0)])
def test_squares64_floats(sq, kind, ctr0, n, nkeys, pad):
    keys = O.keygen(8, nkeys)
    ld = n + pad
    out = getattr(sq, f"fill_{kind}")(_dev_keys(keys), ctr0, n, ld=ld)
    torch.cuda.synchronize()
    want = O.fill(kind, keys, ctr0, n, ld=ld)
    got = out.cpu().numpy()
    assert np.array_equal(got[:, :n].view(np.uint8), want[:, :n].view(np.uint8))
    if nkeys == 1:
        k1 = getattr(sq, f"fill_{kind}_k")(int(keys[0]), ctr0, n)
        torch.cuda.synchronize()
        assert np.array_equal(k1.cpu().numpy().view(np.uint8), want[0, :n].view(np.uint8))


@pytest.mark.parametrize("kind", ["u32", "u64", "f32", "f64", "f32x2"])
@pytest.mark.parametrize("stride", [1, 2, 3, 1 << 32, M64])
def test_strided_fill(sq, kind, stride):
    keys = O.keygen(9, 2)
    ctr0, n = M64 - 12345, 70_001
    out = sq.fill_ex(kind, ctr0, n, stride=stride, keys=_dev_keys(keys))
    torch.cuda.synchronize()
    want = O.fill_strided(kind, keys, ctr0, stride, n)
    got = out.cpu().numpy().reshape(2, -1).view(want.dtype).reshape(2, n) if kind != "f32x2" else \
        out.cpu().numpy().reshape(2, n, 2).view(np.uint64).reshape(2, n)
    assert np.array_equal(got, want), first_mismatch(got.reshape(-1), want.reshape(-1))
    one = sq.fill_ex(kind, ctr0, n, stride=stride, key=int(keys[1]))
    torch.cuda.synchronize()
    g1 = one.cpu().numpy().reshape(-1).view(want.dtype)
    assert np.array_equal(g1, want[1])


def test_fill_ex_rejects_zero_stride(sq):
    with pytest.raises(sq.SquaresError):
        sq.fill_ex("u32", 0, 10, stride=0, key=1)


@pytest.mark.parametrize("kind", ["u32", "u64", "f32", "f64", "f32x2"])
@pytest.mark.parametrize("ctr", [0, 1, 12345, M64])
def test_keyctr(sq, kind, ctr):
    keys = O.keygen(10, 100_003)
    out = sq.fill_keyctr(kind, _dev_keys(keys), ctr)
    torch.cuda.synchronize()
    want = O.fill_keyctr(kind, keys, ctr)
    got = out.cpu().numpy().reshape(-1).view(want.dtype)[: want.size]
    assert np.array_equal(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("kind", ["u32", "u64", "f32", "f64", "f32x2"])
@pytest.mark.parametrize("nkeys,koff,ooff", [(1, 0, 0), (3, 0, 0), (4, 0, 0), (4097, 1, 0), (4098, 0, 1), (70_001, 1, 1)])
def test_keyctr_alignment_and_tails(sq, kind, nkeys, koff, ooff):
    """Key-counter mode's vectorised path (4 keys per thread, 16-byte loads/stores) and its
    per-key fallback: ragged key counts, keys and outputs offset by one element (unaligned)."""
    keys = O.keygen(12, nkeys)
    kbuf = torch.zeros(nkeys + 1, dtype=torch.int64, device="cuda")
    kbuf[koff:koff + nkeys] = _dev_keys(keys)
    es = 8 if kind in ("u64", "f64", "f32x2") else 4
    obuf = torch.full((nkeys + 2,), -1, dtype=torch.int64 if es == 8 else torch.int32, device="cuda")
    dt = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32, "f64": torch.float64, "f32x2": torch.float32}[kind]
    view = obuf[ooff:ooff + nkeys].view(dt)
    if kind == "f32x2":
        view = view.view(nkeys, 2)
    sq.fill_keyctr(kind, kbuf[koff:koff + nkeys], 4242, out=view)
    torch.cuda.synchronize()
    want = O.fill_keyctr(kind, keys, 4242)
    allb = obuf.cpu().numpy().view(np.uint64 if es == 8 else np.uint32)
    got = allb[ooff:ooff + nkeys]
    assert np.array_equal(got, want.reshape(-1).view(got.dtype)[:nkeys]), first_mismatch(got, want)
    assert (allb[:ooff] == allb.dtype.type(-1 & (2 ** (8 * es) - 1))).all()
    assert (allb[ooff + nkeys:] == allb.dtype.type(-1 & (2 ** (8 * es) - 1))).all()


@pytest.mark.parametrize("stride,bitrev", [(1, True), (2, False), (3, True), (1 << 40, False)])
@pytest.mark.parametrize("n", [1000, (1 << 22) + 7])
def test_fused_ex(sq, stride, bitrev, n):
    key = int(O.keygen(1, 1)[0])
    h, o = sq.fused_stats_ex(key, 99, n, stride=stride, bitrev=bitrev)
    torch.cuda.synchronize()
    hw, ow = O.fused_stats_ex(key, 99, stride, n, bitrev)
    assert np.array_equal(h.cpu().numpy().view(np.uint64), hw)
    assert np.array_equal(o.cpu().numpy().view(np.uint64), ow)
