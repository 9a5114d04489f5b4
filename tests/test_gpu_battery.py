"""GPU desk battery (-m gpu): the counts the CUDA kernels produce (fused
histograms of u and of bitrev(u), per-bit ones, bit transitions) equal the counts the oracle
battery takes directly from the oracle's output stream, for identity / bits-reversed /
strided sources; hence the statistics and verdicts agree."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import oracle.battery as OB

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sqb():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200.battery as B
    torch.cuda.set_device(0)
    return B


@pytest.mark.parametrize("stride,bitrev", [(1, False), (1, True), (1 << 32, False), (3, True)])
def test_counts_match_oracle_stream(sqb, stride, bitrev):
    key = int(O.keygen(1, 1)[0])
    ctr0, n = 12345, (1 << 20) + 17
    c = sqb.gpu_counts(key, ctr0, n, stride, bitrev)
    w = O.fill_strided("u32", [key], ctr0, stride, n)[0]
    if bitrev:
        w = np.array([O.bitrev32(int(x)) for x in w], np.uint32)
    oc = OB.counts(w)
    assert np.array_equal(c["hist_hi"], oc["hist_hi"])
    pairs = c["hist_hi"] + c["hist_lo"]
    assert np.array_equal(pairs, oc["pair_hist"])
    assert int(c["ones"].sum()) == oc["ones_total"]
    assert c["transitions"] == oc["transitions"]
    gst = {t.name: t for t in sqb.statistics(c)}
    ost = OB.statistics(oc)
    for name, (stat, p, verdict) in ost.items():
        assert gst[name].verdict == verdict
        assert math.isclose(gst[name].p_value, p, rel_tol=1e-9, abs_tol=1e-12), name


def test_transitions_accumulate_and_split(sqb):
    import paper_2004_06278_b200 as sq
    key = int(O.keygen(2, 1)[0])
    total = sq.transitions(key, 0, 3_000_001)
    # the boundary pair between the two halves is included in a single call only
    a = sq.transitions(key, 0, 1_500_000)
    sq.transitions(key, 1_500_000, 1_500_001, count=a)
    w = O.fill("u32", [key], 1_499_999, 2)[0]
    boundary = ((int(w[0]) >> 31) ^ int(w[1])) & 1
    torch.cuda.synchronize()
    assert int(total.item()) == int(a.item()) + boundary


def test_battery_passes_at_scale(sqb):
    """P:45 "a basic uniformity test ... with no failures", GPU scale: 2^32 outputs."""
    key = int(O.keygen(1, 1)[0])
    res = sqb.run_battery(key, 0, 1 << 32)
    assert all(r.verdict == "pass" for r in res), res
