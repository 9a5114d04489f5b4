"""Pins for the oracle's SURVEY 8(f) functions (-m "not gpu"): squares64-derived floats,
strided counters, key-counter mode and bits-reversed statistics."""
import os
import struct

import numpy as np

import oracle as O
import synth_inputs as SI

M64 = (1 << 64) - 1


def _rows(path):
    out = []
    for line in open(path):
        line = line.split("#", 1)[0].strip()
        if line:
            out.append([int(x, 16) for x in line.split()])
    return out


def _f64_bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _f32_bits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_f64_values(golden_dir):
    for v, bits in _rows(os.path.join(golden_dir, "f64_values.txt")):
        assert _f64_bits(O.f64_from_u64(v)) == bits


def test_f32_pair_examples():
    """raw 0 -> (0, 0); 0x80000000_00000000 -> (0.0, 0.5);
    0x00000000_FFFFFFFF -> ((2^24-1)*2^-24, 0.0) -- low half first."""
    for raw, lo, hi in [(0, 0.0, 0.0), (0x8000000000000000, 0.0, 0.5),
                        (0x00000000FFFFFFFF, (2 ** 24 - 1) * 2.0 ** -24, 0.0)]:
        assert O.f32_from_u32(raw & 0xFFFFFFFF) == lo and O.f32_from_u32(raw >> 32) == hi


def test_f64_and_f32x2_fills_follow_squares64():
    keys = O.keygen(4, 3)
    n = 2000
    u = O.fill("u64", keys, 17, n)
    d = O.fill("f64", keys, 17, n)
    p = O.fill("f32x2", keys, 17, n)
    want_d = ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)      # exact in float64
    assert np.array_equal(d.view(np.uint64), want_d.view(np.uint64))
    lo = ((u & np.uint64(0xFFFFFFFF)) >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
    hi = (u >> np.uint64(40)).astype(np.float64) * 2.0 ** -24
    assert np.array_equal(p[..., 0], lo.astype(np.float32)) and np.array_equal(p[..., 1], hi.astype(np.float32))
    assert d.max() < 1.0 and p.max() < 1.0 and d.min() >= 0.0


def test_strided_reduces_to_fill_and_definition():
    """stride 1 is the ordinary fill; stride 2, n = 2 gives counters c, c + 2."""
    keys = O.keygen(5, 2)
    for kind in ("u32", "u64", "f32", "f64", "f32x2"):
        a = O.fill_strided(kind, keys, 99, 1, 300)
        b = O.fill(kind, keys, 99, 300)
        assert np.array_equal(a.view(np.uint8).reshape(-1), b.view(np.uint8).reshape(-1)), kind
    k = int(keys[0])
    s = O.fill_strided("u32", [k], M64 - 3, 2, 2)[0]
    assert s[0] == O.squares32(M64 - 3, k) and s[1] == O.squares32(M64 - 1, k)
    big = O.fill_strided("u64", [k], 5, 1 << 32, 4)[0]
    assert all(big[i] == O.squares64((5 + i * (1 << 32)) & M64, k) for i in range(4))


def test_keyctr_is_fixed_counter_many_keys():
    """the counter fixed (even 0), the key varies."""
    keys = O.keygen(6, 500)
    for ctr in (0, 12345, M64):
        got = O.fill_keyctr("u32", keys, ctr)
        assert all(got[j] == O.squares32(ctr, int(keys[j])) for j in range(0, 500, 7))
        got64 = O.fill_keyctr("u64", keys, ctr)
        assert all(got64[j] == O.squares64(ctr, int(keys[j])) for j in range(0, 500, 7))


def test_bitrev_examples_and_involution():
    """0x00000001 -> 0x80000000; palindromes fixed; involution."""
    assert O.bitrev32(1) == 0x80000000
    assert O.bitrev32(0x80000001) == 0x80000001
    for u in SI.random_u64(1000, 3).tolist():
        u &= 0xFFFFFFFF
        assert O.bitrev32(O.bitrev32(u)) == u


def test_fused_ex_matches_fill_bitrev_bincount():
    key = int(O.keygen(1, 1)[0])
    n, stride = 1 << 16, 3
    u = O.fill_strided("u32", [key], 7, stride, n)[0]
    r = np.array([O.bitrev32(int(x)) for x in u], dtype=np.uint32)
    for vals, flag in ((u, False), (r, True)):
        h, o = O.fused_stats_ex(key, 7, stride, n, flag)
        assert np.array_equal(h, np.bincount(vals >> np.uint32(16), minlength=65536).astype(np.uint64))
        bits = np.unpackbits(vals.view(np.uint8).reshape(-1, 4), axis=1, bitorder="little").sum(axis=0)
        assert np.array_equal(o, bits.astype(np.uint64))
    # stride 1, no transform == the plain fused statistics
    h1, o1 = O.fused_stats_ex(key, 0, 1, 5000)
    h2, o2 = O.fused_stats(key, 0, 5000)
    assert np.array_equal(h1, h2) and np.array_equal(o1, o2)


def test_scaled_hist_range_pieces_and_chi2():
    """Pieces of the enumeration add up to the whole; the chi-square computed from the whole
    histogram equals oracle.scaled_uniformity's."""
    key, W = 0x5A3B, 16
    whole = O.scaled_hist_range(key, W, 0, 1 << W)
    parts = np.zeros_like(whole)
    for c0 in range(0, 1 << W, 1 << 12):
        O.scaled_hist_range(key, W, c0, 1 << 12, parts)
    assert np.array_equal(whole, parts) and int(whole.sum()) == 1 << W
    e = float(1 << W) / whole.size
    chi2 = float(((whole.astype(np.float64) - e) ** 2).sum() / e)
    assert abs(chi2 - O.scaled_uniformity(key, W)[0]) < 1e-9
    assert O.scaled_hist_range(0, W, 0, 1 << W)[0] == 1 << W
