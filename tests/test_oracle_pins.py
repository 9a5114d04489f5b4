"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it follows (P:n = PAPER.md line n, S:n = SPEC.md line n).  None of
these re-types the oracle's formula: the pins are hand-evaluated values, an analytically
derived closed form, independent multiplications, invariants, special cases and library
routines (numpy.bincount, scipy.special.gammaincc).
"""
import os
import struct

import numpy as np
import pytest

import oracle as O
import synth_inputs as SI

M64 = (1 << 64) - 1


def _read_table(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows


# --------------------------------------------------------------------------- listings
def test_hand_values(golden_dir):
    """Hand-evaluated values of P:21-28 / P:56-64 and SPEC's rot_half/round examples."""
    rows = _read_table(os.path.join(golden_dir, "hand_values.txt"))
    assert len(rows) >= 20
    for fn, a, b, want in rows:
        a, want = int(a, 16), int(want, 16)
        if fn == "squares32":
            assert O.squares32(a, int(b, 16)) == want, (fn, a, b)
        elif fn == "squares64":
            assert O.squares64(a, int(b, 16)) == want, (fn, a, b)
        elif fn == "rot_half":
            assert O.rot_half(a) == want
        elif fn == "round":
            assert O.round_(a, int(b, 16)) == want
        else:
            raise AssertionError(fn)


def _closed_form(c):
    """key = 2^32, 0 <= c <= 1289: derived by hand from the listing.
    Round 1 -> c; round 2 -> c^2*2^32 + (c+1); round 3 -> A*2^32 + B with A = (c+1)^2,
    B = 2c^2(c+1) + c (< 2^32 for c <= 1289); round 4 hi = 2AB + (c+1) + floor(B^2/2^32)."""
    A = (c + 1) ** 2
    B = 2 * c * c * (c + 1) + c
    assert B < 2 ** 32 and A < 2 ** 32
    H = (2 * A * B + (c + 1) + (B * B >> 32)) % 2 ** 32
    L = (B * B) % 2 ** 32
    r5 = (2 * L * H + c + (H * H >> 32)) % 2 ** 32
    return H, (H << 32) | (L ^ r5)


def test_closed_form_key_2_32():
    """Exercises the round-4 lo->hi carry (nonzero from c = 32 on) for both listings."""
    for c in range(0, 1290):
        s32, s64 = _closed_form(c)
        assert O.squares32(c, 1 << 32) == s32, c
        assert O.squares64(c, 1 << 32) == s64, c


def test_three_multiplications_agree():
    """the listing vs two independent 64x64->64 products (16-bit limbs, __int128) on
    10^6 seeded pairs plus the corner cross product."""
    ctr, key = SI.random_pairs(1_000_000)
    for w in (32, 64):
        a = O.squares_pairs(ctr, key, w, "listing")
        b = O.squares_pairs(ctr, key, w, "limb")
        c = O.squares_pairs(ctr, key, w, "i128")
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_python_bignum_transcription_small():
    """A third, arbitrary-precision evaluation on a few thousand pairs (mod 2^64 by hand)."""
    def sq(ctr, key, five):
        m = 2 ** 64
        rot = lambda v: ((v >> 32) | (v << 32)) % m
        y = (ctr * key) % m
        z = (y + key) % m
        x = rot((y * y + y) % m)
        x = rot((x * x + z) % m)
        x = rot((x * x + y) % m)
        if not five:
            return ((x * x + z) % m) >> 32
        t = (x * x + z) % m
        x = rot(t)
        return t ^ (((x * x + y) % m) >> 32)
    ctr, key = SI.random_pairs(3000, seed=5)
    for c, k in zip(ctr.tolist(), key.tolist()):
        assert O.squares32(c, k) == sq(c, k, False)
        assert O.squares64(c, k) == sq(c, k, True)


def test_hi32_of_squares64_is_squares32():
    """P:62-63 vs P:27: round 4 of squares64 keeps t before rotating; the XOR with
    (round5 >> 32) touches only the low half, so hi32(squares64) == squares32 exactly."""
    ctr, key = SI.random_pairs(200_000, seed=11)
    s32 = O.squares_pairs(ctr, key, 32)
    s64 = O.squares_pairs(ctr, key, 64)
    assert np.array_equal((s64 >> np.uint64(32)).astype(np.uint32), s32)


def test_key_zero_gives_zero():
    """key = 0: y = z = 0 and every round stays 0."""
    ctr = SI.random_u64(10_000, seed=3)
    key = np.zeros_like(ctr)
    assert not O.squares_pairs(ctr, key, 32).any()
    assert not O.squares_pairs(ctr, key, 64).any()


def test_weyl_equivalence():
    """(w += s) is equivalent to w = i*s mod 2^64 (10^4 random s, i up to 10^3)."""
    for s in SI.random_u64(10_000, seed=17).tolist() + [0, 1, 3, M64]:
        assert O.weyl_check(s, 1000)
    assert O.weyl_check(3, 6)


def test_determinism_and_rot_involution():
    x = SI.random_u64(1000, seed=23).tolist()
    for v in x:
        assert O.rot_half(O.rot_half(v)) == v
        assert O.squares32(v, 0x123456789ABCDEF3) == O.squares32(v, 0x123456789ABCDEF3)


def test_avalanche_band():
    """one flipped counter bit changes 12..20 of 32 output bits on average."""
    g = np.random.Generator(np.random.PCG64(29))
    ctr, key = SI.random_pairs(100_000, seed=31)
    bit = g.integers(0, 64, size=ctr.size).astype(np.uint64)
    a = O.squares_pairs(ctr, key, 32)
    b = O.squares_pairs(ctr ^ (np.uint64(1) << bit), key, 32)
    ham = np.unpackbits((a ^ b).view(np.uint8)).sum() / a.size
    assert 12.0 <= ham <= 20.0, ham


# --------------------------------------------------------------------------- fills
def test_fill_is_per_counter_definition():
    keys = O.keygen(3, 4)
    ctr0 = M64 - 100          # wraps mod 2^64 inside the range
    n = 300
    out = O.fill("u32", keys, ctr0, n, ld=n + 5)
    out64 = O.fill("u64", keys, ctr0, n, ld=n + 5)
    for k in range(4):
        c = np.array([(ctr0 + i) & M64 for i in range(n)], dtype=np.uint64)
        kk = np.full(n, keys[k], dtype=np.uint64)
        assert np.array_equal(out[k, :n], O.squares_pairs(c, kk, 32))
        assert np.array_equal(out64[k, :n], O.squares_pairs(c, kk, 64))
        assert not out[k, n:].any() and not out64[k, n:].any()   # padding untouched


def test_f32_values(golden_dir):
    """BASELINE.json config 4: top 24 bits of squares32 -> float32 in [0, 1), exact."""
    for u, bits in _read_table(os.path.join(golden_dir, "f32_values.txt")):
        f = O.f32_from_u32(int(u, 16))
        assert struct.unpack("<I", struct.pack("<f", f))[0] == int(bits, 16)


def test_f32_fill_exact_and_in_range():
    keys = O.keygen(7, 3)
    u = O.fill("u32", keys, 0, 5000)
    f = O.fill("f32", keys, 0, 5000)
    # exact: (u >> 8) * 2^-24 computed in float64 (every value is a 24-bit integer times 2^-24)
    want = ((u >> np.uint32(8)).astype(np.float64) * 2.0 ** -24).astype(np.float32)
    assert np.array_equal(f.view(np.uint32), want.view(np.uint32))
    assert f.min() >= 0.0 and f.max() < 1.0


# --------------------------------------------------------------------------- fused stats
def test_fused_key_zero_closed_form():
    """key = 0: every output is 0, so hist[0] = n and every ones count is 0."""
    h, o = O.fused_stats(0, 12345, 100_000)
    assert h[0] == 100_000 and h[1:].sum() == 0 and o.sum() == 0


def test_fused_matches_fill_plus_bincount():
    key = int(O.keygen(1, 1)[0])
    n = 1 << 18
    u = O.fill("u32", [key], 999, n)[0]
    h, o = O.fused_stats(key, 999, n)
    assert np.array_equal(h, np.bincount(u >> np.uint32(16), minlength=65536).astype(np.uint64))
    bits = np.unpackbits(u.view(np.uint8).reshape(-1, 4), axis=1, bitorder="little")  # (n, 32)
    assert np.array_equal(o, bits.sum(axis=0).astype(np.uint64))


def test_fused_invariants_and_additivity():
    key = int(O.keygen(2, 1)[0])
    h, o = O.fused_stats(key, 0, 200_000)
    assert int(h.sum()) == 200_000
    b = np.arange(65536, dtype=np.uint64)
    for j in range(16):   # ones[16+j] = sum of hist over bins with bit j set
        assert int(o[16 + j]) == int(h[(b >> np.uint64(j)) & np.uint64(1) == 1].sum())
    # shards in any order sum to the whole (P:41 counter partitioning)
    hs, os_ = np.zeros(65536, np.uint64), np.zeros(32, np.uint64)
    for start, ln in [(150_000, 50_000), (0, 70_000), (70_000, 80_000)]:
        O.fused_stats(key, start, ln, hs, os_)
    assert np.array_equal(hs, h) and np.array_equal(os_, o)


# --------------------------------------------------------------------------- keys
def test_validate_key_examples():
    """S:156-158 examples and each rule of P:37 / S:136-138."""
    assert O.validate_key(0x123456789ABCDEF3) == 0
    assert O.validate_key(0x113456789ABCDEF3) & O.KEY_UPPER_REPEAT
    assert O.validate_key(0x123456789ABCDEF2) & O.KEY_EVEN
    assert O.validate_key(0x1234567899BCDEF3) & O.KEY_LOWER_REPEAT
    assert O.validate_key(0x023456789ABCDEF3) & O.KEY_ZERO_DIGIT
    assert O.validate_key(0x0) & O.KEY_ZERO_DIGIT
    # popcount: 0x1248124812481241 has 16 ones (digits 1,2,4,8 repeated -> also repeats)
    assert O.validate_key(0x1248124812481241) & O.KEY_POPCOUNT
    # all-ones-heavy key with distinct digits in each half: FEDCBA97 FEDCBA97 -> popcount 48
    assert O.validate_key(0xFEDCBA97FEDCBA97) == O.KEY_POPCOUNT


def test_keygen_rules_distinct_prefix_stable(golden_dir):
    keys = O.keygen(1, 1_000_000)
    assert len(set(keys.tolist())) == keys.size
    v = np.array([O.validate_key(int(k)) for k in keys[:20000]])
    assert not v.any()
    pc = np.unpackbits(keys.view(np.uint8).reshape(-1, 8), axis=1).sum(axis=1)
    assert pc.min() >= 28 and pc.max() <= 36                        # "roughly half ones"
    assert np.array_equal(O.keygen(1, 1000), keys[:1000])           # prefix stability
    assert not np.array_equal(O.keygen(2, 1000), keys[:1000])       # seed matters
    frozen = [int(r[0], 16) for r in _read_table(os.path.join(golden_dir, "keys_seed1.txt"))]
    assert keys[:16].tolist() == frozen
    frozen7 = [int(r[0], 16) for r in _read_table(os.path.join(golden_dir, "keys_seed7.txt"))]
    assert O.keygen(7, 16).tolist() == frozen7


def test_keygen_digit_distribution_is_random_like():
    """P:37 "The digits are also chosen randomly": each digit position uses every allowed digit."""
    keys = O.keygen(5, 20_000)
    d = [(keys >> np.uint64(4 * i)) & np.uint64(15) for i in range(16)]
    for i in range(16):
        vals = np.bincount(d[i].astype(np.int64), minlength=16)
        assert vals[0] == 0
        allowed = [1, 3, 5, 7, 9, 11, 13, 15] if i == 0 else list(range(1, 16))
        assert (vals[allowed] > 0).all()


def test_weak_nonzero_reading_c7():
    """P:39 weak reading: y = ctr*key and z = (ctr+1)*key are never both zero for a
    utility key, because z - y = key != 0."""
    keys = O.keygen(1, 64)
    for k in keys.tolist():
        for c in [0, 1, M64, M64 - 1] + SI.random_u64(200, seed=k & 0xFFFF).tolist():
            y = (c * k) & M64
            z = (y + k) & M64
            assert y != 0 or z != 0


def test_keygen_range_error():
    with pytest.raises(ValueError):
        O.keygen(1, (1 << 31) + 1)


# --------------------------------------------------------------------------- scaled analogue
def test_scaled_w64_equals_squares32():
    ctr, key = SI.random_pairs(100_000, seed=41)
    ref = O.squares_pairs(ctr, key, 32)
    got = np.array([O.squares32_scaled(c, k, 64) for c, k in zip(ctr[:20000].tolist(), key[:20000].tolist())],
                   dtype=np.uint64)
    assert np.array_equal(got.astype(np.uint32), ref[:20000])


def test_scaled_hand_values(golden_dir):
    """Hand-derived W = 8 and W = 16 values (tests/golden/scaled_values.txt, each with its
    derivation): pins the reduced-width masking, the W/2 rotation and the high-half
    extraction below W = 64, where equality with squares32 does not reach."""
    n = 0
    with open(os.path.join(golden_dir, "scaled_values.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            W, ctr, key, want = line.split()
            assert O.squares32_scaled(int(ctr, 16), int(key, 16), int(W)) == int(want, 16), line
            n += 1
    assert n == 8


def test_scaled_key_zero_constant():
    assert all(O.squares32_scaled(c, 0, 16) == 0 for c in range(1 << 16))


def _scaled_key(g, W):
    """A rule-valid W-bit key: distinct nonzero hex digits in each half, d0 odd."""
    nd = W // 4
    half = nd // 2
    up = g.choice(np.arange(1, 16), size=half, replace=False)
    d0 = g.choice(np.arange(1, 16, 2))
    rest = g.choice([d for d in range(1, 16) if d != d0], size=half - 1, replace=False)
    digits = [int(d0)] + [int(x) for x in rest] + [int(x) for x in up]
    return sum(d << (4 * i) for i, d in enumerate(digits))


def test_scaled_uniformity_w16():
    """exhaustive W = 16 for 10 rule-valid scaled keys; >= 9 of 10 p-values > 1e-4."""
    g = np.random.Generator(np.random.PCG64(53))
    ps = [O.scaled_uniformity(_scaled_key(g, 16), 16)[1] for _ in range(10)]
    assert sum(p > 1e-4 for p in ps) >= 9, ps


def test_gammaq_against_scipy():
    """chi-square p-values at df 255 and 65535 vs an independent evaluation."""
    sp = pytest.importorskip("scipy.special")
    for df in (15, 255, 4095, 65535):
        for z in (-3.0, -1.0, 0.0, 1.5, 4.0):
            x = df + z * np.sqrt(2 * df)
            if x <= 0:
                continue
            want = sp.gammaincc(df / 2, x / 2)
            got = O.gammaq(df / 2, x / 2)
            assert abs(got - want) <= 1e-9 + 1e-7 * abs(want), (df, z, got, want)


# --------------------------------------------------------------------------- partition
def test_partition_examples_and_coverage():
    """S:290-292 examples; disjointness and coverage in wide arithmetic."""
    assert O.partition(1 << 64, 1, 0) == (0, 1 << 64)
    assert O.partition(1 << 64, 2, 1) == (1 << 63, 1 << 63)
    s, ln = O.partition(1 << 64, 10 ** 7, 123)
    assert abs(ln - 1.844674e12) < 1e6                                 # P:41 "about 1.8 trillion"
    for n in [0, 1, 7, 1 << 30, (1 << 38) + 5, 1 << 64]:
        for parts in [1, 2, 3, 8, 1000]:
            pos = 0
            for i in range(parts):
                st, ln = O.partition(n, parts, i)
                assert st == pos
                pos += ln
            assert pos == n
    with pytest.raises(ValueError):
        O.partition(10, 0, 0)


def test_xorfold_u32():
    """oracle_xorfold_u32 (the CPU baseline's dead-code guard): XOR over i of
    squares32(ctr0 + i) << (i mod 32).  Pinned by the hand value squares32(1, 2^32) = 0x2a
    (n = 1), key 0 -> 0, n = 0 -> 0, and by the same fold of the per-element fill done in numpy
    (a different loop: whole-array shifts and a reduction)."""
    assert O.xorfold_u32(1 << 32, 1, 1) == 0x2A
    assert O.xorfold_u32(0, 123, 1000) == 0
    assert O.xorfold_u32(0x123456789ABCDEF3, 5, 0) == 0
    key = int(O.keygen(1, 1)[0])
    for ctr0, n in [(0, 1 << 16), ((1 << 64) - 100, 333), ((1 << 32) - 7, 64)]:
        u = O.fill("u32", [key], ctr0, n)[0].astype(np.uint64)
        sh = (np.arange(n, dtype=np.uint64) & np.uint64(31))
        want = int(np.bitwise_xor.reduce(u << sh)) if n else 0
        assert O.xorfold_u32(key, ctr0, n) == want
