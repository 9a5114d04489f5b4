"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact for every u32/u64 output, every float32 (a
deterministic integer->float map) and every count.  Inputs are seeded and synthetic
(synth_inputs.py); keys come from the ORACLE's key utility so no oracle input is produced by the
product.  Sizes: small cases span several warp chunks and ragged tails; the full-size configs of
BASELINE.json (c2, c3, c4) are compared in full against the oracle run on all host cores; c5
(2^38 counters) is checked by invariants plus oracle parity on sampled sub-ranges, and its first
2^36 counters (all 2^38 with SQ_FULL_ORACLE=1) against the oracle over the whole range.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth_inputs as SI
from tests.helpers import first_mismatch, par_fill, par_fused

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
VIEW = {"u32": np.uint32, "u64": np.uint64, "f32": np.uint32}


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    torch.cuda.set_device(0)
    return sq


def _dev_keys(keys_np):
    return torch.from_numpy(np.ascontiguousarray(keys_np, dtype=np.uint64).view(np.int64)).cuda()


def _bits(t: torch.Tensor, kind):
    return t.cpu().numpy().view(VIEW[kind])


# ----------------------------------------------------------------------------- fills, small
@pytest.mark.parametrize("kind", ["u32", "u64", "f32"])
def test_fill_c1_full(sq, kind):
    """BASELINE.json config 1 shape (2^20 counters, key from seed 1) for every kind."""
    key = int(O.keygen(1, 1)[0])
    out = getattr(sq, f"fill_{kind}")(_dev_keys([key]), 0, 1 << 20)
    torch.cuda.synchronize()
    got = _bits(out, kind)[0]
    want = O.fill(kind, [key], 0, 1 << 20)[0].view(VIEW[kind])
    assert np.array_equal(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("kind", ["u32", "u64", "f32"])
@pytest.mark.parametrize("edge", SI.FILL_EDGES)
def test_fill_edges(sq, kind, edge):
    """n = 0/1/3/5, counter wrap at 2^64, 32-bit counter carry, ragged tails, misaligned output
    pointer, multi-key rows with padding (sentinel check: padding must stay untouched)."""
    ctr0, n, nkeys, ld_pad, off = edge
    keys = O.keygen(11, nkeys)
    ld = n + ld_pad
    es = 8 if kind == "u64" else 4
    dt = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32}[kind]
    total = off + nkeys * ld + 64
    sentinel = torch.full((total,), -1, dtype=torch.int32 if es == 4 else torch.int64).view(dt).cuda()
    view = sentinel[off: off + nkeys * ld]
    getattr(sq, f"fill_{kind}")(_dev_keys(keys), ctr0, n, out=view, ld=ld)
    torch.cuda.synchronize()
    allbits = sentinel.cpu().numpy().view(VIEW[kind])
    fill_val = VIEW[kind](-1 & (M64 if es == 8 else 0xFFFFFFFF))
    want = O.fill(kind, keys, ctr0, n, ld=ld).view(VIEW[kind])
    got = allbits[off: off + nkeys * ld].reshape(nkeys, ld) if nkeys * ld else np.zeros((nkeys, 0), VIEW[kind])
    for k in range(nkeys):
        assert np.array_equal(got[k, :n], want[k, :n]), (k, first_mismatch(got[k, :n], want[k, :n]))
        assert (got[k, n:] == fill_val).all(), "padding between rows was written"
    assert (allbits[:off] == fill_val).all() and (allbits[off + nkeys * ld:] == fill_val).all()


@pytest.mark.parametrize("kind", ["u32", "u64", "f32"])
@pytest.mark.parametrize("ctr0,n", [(0, 1), (7, 33), ((1 << 64) - 1000, 4099), ((1 << 32) - 5, (1 << 20) + 17)])
def test_fill_by_value_key(sq, kind, ctr0, n):
    """sq_fill_*_k (key by value, uniform-register constants) vs the oracle, incl. a
    misaligned output pointer (offset by one element)."""
    key = int(O.keygen(2, 1)[0])
    dt = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32}[kind]
    buf = torch.zeros(n + 2, dtype=dt, device="cuda")
    getattr(sq, f"fill_{kind}_k")(key, ctr0, n, out=buf[1:n + 1])
    torch.cuda.synchronize()
    got = buf.cpu().numpy().view(VIEW[kind])
    want = O.fill(kind, [key], ctr0, n)[0].view(VIEW[kind])
    assert np.array_equal(got[1:n + 1], want), first_mismatch(got[1:n + 1], want)
    assert got[0] == 0 and got[n + 1] == 0


@pytest.mark.parametrize("kind", ["u32", "u64"])
def test_fill_corner_keys(sq, kind):
    """Kernels are total over (ctr, key): key 0, 1, 2^32, 2^64-1 and random odd/even."""
    keys = np.array([0, 1, 1 << 32, M64, 0x123456789ABCDEF3] + SI.random_u64(3, 5).tolist(), dtype=np.uint64)
    for ctr0 in (0, (1 << 32) - 100, M64 - 300):
        out = getattr(sq, f"fill_{kind}")(_dev_keys(keys), ctr0, 777)
        torch.cuda.synchronize()
        got = _bits(out, kind)
        want = O.fill(kind, keys, ctr0, 777).view(VIEW[kind])
        assert np.array_equal(got, want)


def test_fill_random_pairs(sq):
    """Fuzz: seeded random (ctr, key) pairs plus the full corner cross product, each evaluated
    as a short fill row starting at that counter (so the state initialisation at an arbitrary
    counter and the first steps are exercised for every pair)."""
    ctr, key = SI.random_pairs(2000, seed=SI.FUZZ_SEED)
    for j in range(ctr.size):
        c, k = int(ctr[j]), int(key[j])
        o32 = _bits(sq.fill_u32(_dev_keys([k]), c, 3), "u32")[0]
        o64 = _bits(sq.fill_u64(_dev_keys([k]), c, 3), "u64")[0]
        for i in range(3):
            assert o32[i] == O.squares32((c + i) & M64, k), (hex(c), hex(k), i)
            assert o64[i] == O.squares64((c + i) & M64, k), (hex(c), hex(k), i)


def test_gpu_hi32_of_u64_equals_u32(sq):
    """P:62-63 vs P:27 on the GPU outputs themselves."""
    keys = _dev_keys(O.keygen(3, 2))
    a = sq.fill_u32(keys, 5, 100_003)
    b = sq.fill_u64(keys, 5, 100_003)
    torch.cuda.synchronize()
    assert np.array_equal((_bits(b, "u64") >> np.uint64(32)).astype(np.uint32), _bits(a, "u32"))


def test_fill_stream_semantics(sq):
    """Asynchronous on the caller's stream: a side stream's result is visible after its sync."""
    s = torch.cuda.Stream()
    keys = _dev_keys(O.keygen(1, 1))
    with torch.cuda.stream(s):
        out = sq.fill_u32(keys, 0, 1 << 16)
    s.synchronize()
    want = O.fill("u32", O.keygen(1, 1), 0, 1 << 16)
    assert np.array_equal(_bits(out, "u32"), want)


# ----------------------------------------------------------------------------- fills, full size
@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_fill_full_size_single_key(sq, cfg):
    """BASELINE.json configs 2 and 3 at full size (4 GiB each), compared in full through BOTH
    entry points: sq_fill_u32/u64 (device key array, the 8(b) call) and sq_fill_u32_k/u64_k
    (key by value: the kernel instantiation bench.py times, with its own register allocation)."""
    w = SI.CONFIGS[cfg]
    key = int(O.keygen(w.key_seed, 1)[0])
    want = par_fill(w.kind, key, w.ctr0, w.n).view(VIEW[w.kind])
    out = getattr(sq, f"fill_{w.kind}")(_dev_keys([key]), w.ctr0, w.n)
    torch.cuda.synchronize()
    got = _bits(out, w.kind)[0]
    assert np.array_equal(got, want), first_mismatch(got, want)
    out.fill_(-1)   # the by-value run must write every element itself
    getattr(sq, f"fill_{w.kind}_k")(key, w.ctr0, w.n, out=out.view(-1))
    torch.cuda.synchronize()
    got = _bits(out, w.kind)[0]
    del out
    torch.cuda.empty_cache()
    assert np.array_equal(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("kind", ["u32", "u64"])
def test_fill_beyond_2_32_elements(sq, kind):
    """Maximum-size edge: one row of 2^32 + 1000 elements (16/32 GiB) starting 2^31 counters
    before the 2^64 wrap, through the key-by-value entry point bench.py times.  Every element
    index and byte offset passes 2^32; checked against the oracle's pair evaluator on the first
    and last 2^20 elements, 2^20 random ones and the elements around the wrap."""
    key = int(O.keygen(1, 1)[0])
    n = (1 << 32) + 1000
    ctr0 = (1 << 64) - (1 << 31)
    es = 8 if kind == "u64" else 4
    out = torch.empty(n, dtype=torch.int32 if es == 4 else torch.int64, device="cuda")
    getattr(sq, f"fill_{kind}_k")(key, ctr0, n, out=out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(20040627)
    idx = np.unique(np.concatenate([np.arange(1 << 20), np.arange(n - (1 << 20), n),
                                    rng.integers(0, n, 1 << 20), np.arange((1 << 31) - 8, (1 << 31) + 8)]))
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint32 if es == 4 else np.uint64)
    ctr = (np.uint64(ctr0) + idx.astype(np.uint64))   # wraps mod 2^64 in uint64 arithmetic
    want = O.squares_pairs(ctr, np.full(idx.shape, key, dtype=np.uint64), width=32 if es == 4 else 64)
    assert np.array_equal(got, want), first_mismatch(got, want)
    del out
    torch.cuda.empty_cache()


def test_fill_full_size_c4(sq):
    """BASELINE.json config 4: 4096 keys (seed 7) x 2^18 counters as float32, [key][ctr]."""
    w = SI.CONFIGS["c4"]
    keys = O.keygen(w.key_seed, w.nkeys)
    out = sq.fill_f32(_dev_keys(keys), w.ctr0, w.n)
    torch.cuda.synchronize()
    got = _bits(out, "f32")
    del out
    from concurrent.futures import ThreadPoolExecutor
    from tests.helpers import ncores
    with ThreadPoolExecutor(ncores()) as ex:
        rows = list(ex.map(lambda k: O.fill("f32", [int(k)], w.ctr0, w.n)[0], keys))
    want = np.stack(rows).view(np.uint32)
    assert np.array_equal(got, want), first_mismatch(got.reshape(-1), want.reshape(-1))
    f = got.view(np.float32)
    assert f.min() >= 0.0 and f.max() < 1.0


# ----------------------------------------------------------------------------- fused statistics
def _fused(sq, key, ctr0, n):
    h, o = sq.fused_stats(key, ctr0, n)
    torch.cuda.synchronize()
    return h.cpu().numpy().view(np.uint64), o.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 1000, 32768 * 3 + 7, (1 << 20) + 5, 1 << 22])
def test_fused_small(sq, n):
    key = int(O.keygen(1, 1)[0])
    h, o = _fused(sq, key, 77, n)
    hw, ow = O.fused_stats(key, 77, n)
    assert np.array_equal(h, hw), first_mismatch(h, hw)
    assert np.array_equal(o, ow), first_mismatch(o, ow)


def test_fused_accumulates(sq):
    key = int(O.keygen(1, 1)[0])
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    o = torch.zeros(32, dtype=torch.int64, device="cuda")
    for start, ln in [(0, 100_000), (100_000, 1 << 20), (100_000 + (1 << 20), 12345)]:
        sq.fused_stats(key, start, ln, h, o)
    torch.cuda.synchronize()
    hw, ow = O.fused_stats(key, 0, 100_000 + (1 << 20) + 12345)
    assert np.array_equal(h.cpu().numpy().view(np.uint64), hw)
    assert np.array_equal(o.cpu().numpy().view(np.uint64), ow)


def test_fused_key_zero_guard_path(sq):
    """key = 0: every sample lands in bin 0, so the shared-memory histogram is swept to global
    memory at almost every epoch barrier (hist16.cuh sweep scheme); closed form hist[0] = n,
    ones = 0."""
    n = 1 << 26
    h, o = _fused(sq, 0, 5, n)
    assert h[0] == n and h[1:].sum() == 0 and o.sum() == 0


def test_fused_hot_bins_both_halves(sq):
    """key = 2^32: outputs concentrate on few bins for small counters (closed form family);
    checks sweeps of hot bins in both 16-bit halves against the oracle."""
    n = 1 << 23
    h, o = _fused(sq, 1 << 32, 0, n)
    hw, ow = O.fused_stats(1 << 32, 0, n)
    assert np.array_equal(h, hw) and np.array_equal(o, ow)


@pytest.mark.parametrize("key", [1 << 32, (1 << 32) + (1 << 16)])
def test_fused_hot_bins_accumulate_in_pieces(sq, key):
    """Hot bins (closed-form key family) counted in three pieces into the same non-zero arrays:
    the sweeps of each piece (A/B word packing of hist16.cuh, derived ones[16..31]) must add up
    to the single-run oracle."""
    n = (1 << 23) + 12345
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    o = torch.zeros(32, dtype=torch.int64, device="cuda")
    cuts = [0, 1 << 21, (1 << 21) + 777, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        sq.fused_stats(key, 3 + a, b - a, h, o)
    torch.cuda.synchronize()
    hw, ow = O.fused_stats(key, 3, n)
    assert np.array_equal(h.cpu().numpy().view(np.uint64), hw)
    assert np.array_equal(o.cpu().numpy().view(np.uint64), ow)


def test_fused_sweeps_at_scale(sq):
    """Many sweeps per CTA: key = 2^32 (outputs concentrated on few bins for small counters,
    closed-form family) over 2^30 counters vs the parallel oracle, and key = 0 over 2^32
    counters (every sample in bin 0: a sweep at almost every epoch barrier) vs its closed form."""
    n = 1 << 30
    h, o = _fused(sq, 1 << 32, 0, n)
    hw, ow = par_fused(1 << 32, 0, n)
    assert np.array_equal(h, hw), first_mismatch(h, hw)
    assert np.array_equal(o, ow), first_mismatch(o, ow)
    n0 = 1 << 32
    h0, o0 = _fused(sq, 0, 12345, n0)
    assert int(h0[0]) == n0 and int(h0[1:].sum()) == 0 and int(o0.sum()) == 0


def test_fused_2_30_vs_parallel_oracle(sq):
    key = int(O.keygen(1, 1)[0])
    n = 1 << 30
    h, o = _fused(sq, key, 0, n)
    hw, ow = par_fused(key, 0, n)
    assert np.array_equal(h, hw), first_mismatch(h, hw)
    assert np.array_equal(o, ow), first_mismatch(o, ow)


def test_fused_c5_full_size(sq):
    """BASELINE.json config 5 (2^38 counters, one GPU): invariants at full size, and oracle
    parity on sampled sub-ranges (the fused map is additive over counter ranges)."""
    w = SI.CONFIGS["c5"]
    key = int(O.keygen(w.key_seed, 1)[0])
    h, o = _fused(sq, key, w.ctr0, w.n)
    assert int(h.sum()) == w.n
    b = np.arange(65536, dtype=np.uint64)
    for j in range(16):
        assert int(o[16 + j]) == int(h[(b >> np.uint64(j)) & np.uint64(1) == 1].sum())
    # plausibility bands (not parity): E[hist] = 2^22, sd ~ 2^11; E[ones] = 2^37, sd = 2^18
    assert abs(h.astype(np.float64).mean() - 2 ** 22) < 1
    assert np.abs(h.astype(np.float64) - 2 ** 22).max() < 12 * 2 ** 11
    assert np.abs(o.astype(np.float64) - 2 ** 37).max() < 8 * 2 ** 18
    # sampled sub-ranges at the start, the middle and the end of the counter range
    for start in (0, (1 << 37) + 12345, w.n - (1 << 24)):
        hs, os_ = _fused(sq, key, start, 1 << 24)
        hw, ow = par_fused(key, start, 1 << 24)
        assert np.array_equal(hs, hw) and np.array_equal(os_, ow), start


def test_fused_c5_vs_full_oracle(sq):
    """BASELINE.json config 5 against the oracle run over a WHOLE counter range on all host
    cores, every histogram bin and every per-bit count bit-exact: by default the first 2^36
    counters of c5 (a quarter of the config, ~85 s of 16 host cores, launched exactly as the
    bench launches c5: one call over the range); SQ_FULL_ORACLE=1 compares the full 2^38
    (337 s on the 16-core GPU host; log: profiles/r01_c5_full_oracle_pytest.log)."""
    w = SI.CONFIGS["c5"]
    n = w.n if os.environ.get("SQ_FULL_ORACLE") == "1" else 1 << 36
    key = int(O.keygen(w.key_seed, 1)[0])
    h, o = _fused(sq, key, w.ctr0, n)
    hw, ow = par_fused(key, w.ctr0, n)
    assert np.array_equal(h, hw), first_mismatch(h, hw)
    assert np.array_equal(o, ow), first_mismatch(o, ow)


def test_fill_host_e2e(sq):
    """sq_fill_host: chunked generate + D2H into pinned host memory equals the oracle."""
    key = int(O.keygen(1, 1)[0])
    n = (1 << 22) + 3
    scratch = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    for kind in ("u32", "u64", "f32"):
        es = 8 if kind == "u64" else 4
        host = torch.empty(n * es, dtype=torch.uint8).pin_memory()
        sq.fill_host(kind, key, 99, n, host, scratch, copy_stream=torch.cuda.Stream())
        got = host.numpy().view(VIEW[kind])
        want = O.fill(kind, [key], 99, n)[0].view(VIEW[kind])
        assert np.array_equal(got, want), (kind, first_mismatch(got, want))


@pytest.mark.parametrize("kind", ["u32", "u64", "f32", "f64", "f32x2"])
@pytest.mark.parametrize("scratch_bytes,n,ctr0", [(64, 1000, 5), (100, 4097, (1 << 64) - 700), (3 << 20, (1 << 21) + 9, 1 << 40)])
def test_fill_host_chunking(sq, kind, scratch_bytes, n, ctr0):
    """sq_fill_host with tiny and odd scratch sizes (chunks of one or a few 32-byte halves, ragged
    last chunk, the counter wrap inside the range) and pageable as well as pinned host memory."""
    key = int(O.keygen(2, 1)[0])
    es = 8 if kind in ("u64", "f64", "f32x2") else 4
    for pinned in (True, False):
        host = torch.zeros(n * es + 16, dtype=torch.uint8)
        if pinned:
            host = host.pin_memory()
        scratch = torch.empty(scratch_bytes, dtype=torch.uint8, device="cuda")
        sq.fill_host(kind, key, ctr0, n, host, scratch)
        want = O.fill_strided(kind, [key], ctr0, 1, n)[0]
        got = host.numpy()[: n * es].view(want.dtype)
        assert np.array_equal(got, want), (kind, pinned, first_mismatch(got, want))
        assert (host.numpy()[n * es:] == 0).all()


def test_parity_harness_detects_a_flipped_word(sq):
    """Negative test (failure detection): the comparison used throughout this file
    must fail, and name the first bad index, when one output word or one count is wrong."""
    key = int(O.keygen(1, 1)[0])
    n = (1 << 16) + 3
    out = sq.fill_u32_k(key, 0, n)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32).copy()
    want = O.fill("u32", [key], 0, n)[0]
    assert np.array_equal(got, want)
    for i in (0, 12345, n - 1):
        bad = got.copy()
        bad[i] ^= np.uint32(1 << (i % 32))
        assert not np.array_equal(bad, want)
        assert first_mismatch(bad, want).startswith(f"1 mismatches; first at {i}:")
    h, o = _fused(sq, key, 0, n)
    hw, ow = O.fused_stats(key, 0, n)
    assert np.array_equal(h, hw) and np.array_equal(o, ow)
    h2 = h.copy()
    h2[int(np.argmax(h2))] += np.uint64(1)
    assert not np.array_equal(h2, hw)
