"""Pins of the oracle desk battery (oracle/battery.py) on constructed streams, following SPEC's
examples, and the paper's claim that squares passes a basic uniformity test
at desk scale for utility keys, including bits-reversed and stride-2^32 sources."""
import numpy as np
import pytest

import oracle as O
import oracle.battery as B


def test_all_zero_stream_fails():
    """an all-zero source fails (monobit p ~ 0)."""
    st = B.statistics(B.counts(np.zeros(1 << 16, np.uint32)))
    assert st["monobit"][2] == "fail" and st["monobit"][1] < 1e-100
    assert st["byte_chi_square"][2] == "fail" and st["serial_pair"][2] == "fail"
    assert st["runs"][2] == "dependent-failure"


def test_balanced_bits_statistic_zero():
    """exactly balanced bits -> statistic 0, p = 1."""
    st = B.statistics(B.counts(np.full(1 << 14, 0x0F0F0F0F, np.uint32)))
    assert st["monobit"][0] == 0.0 and st["monobit"][1] == 1.0


def test_byte_chi_square_perfect_fit():
    """bytes 0..255 repeated exactly -> statistic 0 (p = 1: fails the two-sided
    verdict, as too perfect a fit should)."""
    w = np.arange(256, dtype=np.uint8).repeat(1).reshape(1, 256).repeat(256, axis=0).reshape(-1).view(np.uint32)
    st = B.statistics(B.counts(w))
    assert st["byte_chi_square"][0] == 0.0 and st["byte_chi_square"][1] == 1.0


def test_serial_pair_degenerate_and_perfect():
    """alternating 0x00, 0x01 bytes load one pair bin -> fail; exact uniform pair
    coverage -> statistic 0."""
    w = np.tile(np.array([0, 1], np.uint8), 1 << 16).view(np.uint32)
    assert B.statistics(B.counts(w))["serial_pair"][2] == "fail"
    w2 = np.arange(65536, dtype=np.uint16).view(np.uint32)
    assert B.statistics(B.counts(w2))["serial_pair"][0] == 0.0


def test_runs_extremes():
    """alternating bits 0101... -> fail (too many runs); all ones -> dependent failure."""
    st = B.statistics(B.counts(np.full(1 << 14, 0x55555555, np.uint32)))
    assert st["runs"][2] == "fail"
    st1 = B.statistics(B.counts(np.full(1 << 14, 0xFFFFFFFF, np.uint32)))
    assert st1["runs"][2] == "dependent-failure"


def test_counts_against_definitions():
    w = np.array([0x00000001, 0x80000000, 0xFFFF0000], np.uint32)
    c = B.counts(w)
    # bits LSB-first: 1,0*31 | 0*31,1 | 0*16,1*16 -> transitions: 1 + 1 (bit31 of w1=1 vs bit0 of w2=0) ... count directly
    bits = [(int(x) >> j) & 1 for x in w for j in range(32)]
    assert c["transitions"] == sum(bits[i] != bits[i + 1] for i in range(len(bits) - 1))
    assert c["ones_total"] == sum(bits)


@pytest.mark.parametrize("source", ["identity", "bitrev", "stride32"])
def test_squares32_passes_desk_battery(source):
    """squares passes a basic uniformity test (desk scale: 2^22 outputs, alpha 1e-6)."""
    key = int(O.keygen(1, 1)[0])
    n = 1 << 22
    if source == "stride32":
        w = O.fill_strided("u32", [key], 0, 1 << 32, n)[0]
    else:
        w = O.fill("u32", [key], 0, n)[0]
        if source == "bitrev":
            w = np.array([O.bitrev32(int(x)) for x in w[: 1 << 18]], np.uint32)
    st = B.statistics(B.counts(w))
    assert all(v[2] == "pass" for v in st.values()), st
