"""Host-side tests of libsquares.so (-m "not gpu"): the library loads, exports every symbol
include/squares.h declares, its host functions agree with the oracle, and the GPU entry points
reject bad arguments before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import synth_inputs as SI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    return sq


def _declared_functions():
    txt = open(os.path.join(ROOT, "include", "squares.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(sq_\w+)\s*\(", txt, flags=re.M)))


def test_header_symbols_exported(sq):
    names = _declared_functions()
    assert len(names) >= 10, names
    lib = ctypes.CDLL(sq.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/squares.h but not exported"
    assert set(names) == set(sq.EXPORTED_SYMBOLS)


def test_version_and_strerror(sq):
    lib = sq._load()
    assert sq.version() >= 100
    for c in range(5):
        assert lib.sq_strerror(c)
    assert lib.sq_strerror(99)


def test_validate_key_matches_oracle(sq):
    keys = SI.random_u64(20000, seed=71).tolist() + [0x123456789ABCDEF3, 0x113456789ABCDEF3,
                                                      0x123456789ABCDEF2, 0, (1 << 64) - 1]
    keys += O.keygen(9, 2000).tolist()
    for k in keys:
        assert sq.validate_key(k) == O.validate_key(k), hex(k)


def test_keygen_matches_oracle(sq):
    for seed, count in [(1, 1), (1, 5000), (7, 4096), (123456789, 300), ((1 << 64) - 1, 50)]:
        got = sq.keygen(seed, count).numpy().view(np.uint64)
        want = O.keygen(seed, count)
        assert np.array_equal(got, want), seed
    assert sq.keygen(3, 0).numel() == 0


def test_keygen_range_error(sq):
    with pytest.raises(sq.SquaresError):
        sq.keygen(1, (1 << 31) + 1)
    assert sq._load().sq_keygen(1, 5, None) == sq.SQ_EINVAL


def test_fill_argument_errors_without_device(sq):
    """Argument checks happen before any CUDA call, so they run on a CPU-only box."""
    lib = sq._load()
    fake_keys, fake_out = 0x10000, 0x20000
    for fn in (lib.sq_fill_u32, lib.sq_fill_u64, lib.sq_fill_f32):
        assert fn(fake_keys, 1, 0, 0, fake_out, 0, None) == sq.SQ_OK        # n == 0: no-op
        assert fn(fake_keys, 0, 0, 100, fake_out, 100, None) == sq.SQ_OK    # nkeys == 0: no-op
        assert fn(None, 1, 0, 10, fake_out, 10, None) == sq.SQ_EINVAL
        assert fn(fake_keys, 1, 0, 10, None, 10, None) == sq.SQ_EINVAL
        assert fn(fake_keys, 2, 0, 10, fake_out, 9, None) == sq.SQ_EINVAL    # ld < n
        assert fn(fake_keys, 1, 0, 10, fake_out + 2, 10, None) == sq.SQ_EINVAL  # misaligned
        assert fn(fake_keys, 1 << 40, 0, 1 << 40, fake_out, 1 << 40, None) == sq.SQ_EINVAL  # size
    for fn in (lib.sq_fill_u32_k, lib.sq_fill_u64_k, lib.sq_fill_f32_k):
        assert fn(1, 0, 0, None, None) == sq.SQ_OK
        assert fn(1, 0, 10, None, None) == sq.SQ_EINVAL
        assert fn(1, 0, 10, fake_out + 2, None) == sq.SQ_EINVAL
    assert lib.sq_fused_stats(1, 0, 0, None, None, None) == sq.SQ_OK
    assert lib.sq_fused_stats(1, 0, 5, None, 0x1000, None) == sq.SQ_EINVAL
    assert lib.sq_fused_stats(1, 0, 5, 0x1004, 0x1000, None) == sq.SQ_EINVAL
    assert lib.sq_fill_host(7, 1, 0, 5, 0x1000, 0x2000, 4096, None, None) == sq.SQ_EINVAL
    assert lib.sq_fill_host(0, 1, 0, 0, None, None, 0, None, None) == sq.SQ_OK
    assert lib.sq_fill_host(0, 1, 0, 5, 0x1000, 0x2000, 16, None, None) == sq.SQ_EINVAL


def test_extended_entry_points_argument_errors_without_device(sq):
    """The 8(f) entry points validate before any CUDA call (CPU-only box): bad kind / stride /
    flags / width / alignment -> SQ_EINVAL, empty work -> SQ_OK, too many keys -> SQ_ERANGE."""
    lib = sq._load()
    K, O_, H, C = 0x10000, 0x20000, 0x30000, 0x40000
    # sq_fill_ex(kind, keys, nkeys, key_imm, ctr0, stride, n, out, ld, stream)
    assert lib.sq_fill_ex(9, K, 1, 0, 0, 1, 10, O_, 10, None) == sq.SQ_EINVAL          # kind
    assert lib.sq_fill_ex(0, K, 1, 0, 0, 0, 10, O_, 10, None) == sq.SQ_EINVAL          # stride 0
    assert lib.sq_fill_ex(0, None, 2, 7, 0, 1, 10, O_, 10, None) == sq.SQ_EINVAL       # by value, 2 rows
    assert lib.sq_fill_ex(1, K, 1, 0, 0, 1, 10, O_ + 4, 10, None) == sq.SQ_EINVAL      # u64 misaligned
    assert lib.sq_fill_ex(0, K, 1, 0, 0, 3, 0, O_, 0, None) == sq.SQ_OK                # n == 0
    # sq_fill_keyctr(kind, keys, nkeys, ctr, out, stream)
    assert lib.sq_fill_keyctr(0, K, 0, 5, O_, None) == sq.SQ_OK
    assert lib.sq_fill_keyctr(0, None, 3, 5, O_, None) == sq.SQ_EINVAL
    assert lib.sq_fill_keyctr(0, K + 4, 3, 5, O_, None) == sq.SQ_EINVAL                # keys misaligned
    assert lib.sq_fill_keyctr(5, K, 3, 5, O_, None) == sq.SQ_EINVAL                    # kind
    # sq_fused_stats_ex(key, ctr0, stride, n, flags, hist, ones, stream)
    assert lib.sq_fused_stats_ex(1, 0, 0, 5, 0, H, H, None) == sq.SQ_EINVAL            # stride 0
    assert lib.sq_fused_stats_ex(1, 0, 1, 5, 2, H, H, None) == sq.SQ_EINVAL            # unknown flag
    assert lib.sq_fused_stats_ex(1, 0, 1, 0, 1, None, None, None) == sq.SQ_OK
    # sq_transitions(key, ctr0, stride, n, flags, count, stream)
    assert lib.sq_transitions(1, 0, 1, 5, 0, C + 4, None) == sq.SQ_EINVAL              # misaligned
    assert lib.sq_transitions(1, 0, 1, 0, 0, None, None) == sq.SQ_OK
    # sq_scaled_hist(W, keys, nkeys, hist, stream)
    for W in (6, 9, 34):
        assert lib.sq_scaled_hist(W, K, 1, H, None) == sq.SQ_EINVAL
    assert lib.sq_scaled_hist(16, K, 0, H, None) == sq.SQ_OK
    assert lib.sq_scaled_hist(16, K, 65536, H, None) == sq.SQ_ERANGE


def test_product_never_imports_oracle():
    """The product path must not reference the oracle (checked textually)."""
    pkg = os.path.join(ROOT, "paper_2004_06278_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle." not in txt.replace("oracle/oracle.c", ""), f
                assert "liboracle" not in txt, f
