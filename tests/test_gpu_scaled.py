"""GPU exhaustive reduced-width uniformity (-m gpu, SPEC S:381-389, P:17 footnote
1): sq_scaled_hist histograms equal the oracle's exhaustive enumeration for W = 8..24 and for
W = 32 (one key, oracle run in parallel shards); key 0 drives all 2^32 counts into one bin (the
histogram sweep path); and at W = 32, >= 90 % of 32 rule-valid scaled keys give p > 1e-4."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import ncores

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    torch.cuda.set_device(0)
    return sq


def _scaled_key(g, W):
    nd = W // 4
    half = nd // 2
    up = g.choice(np.arange(1, 16), size=half, replace=False)
    d0 = g.choice(np.arange(1, 16, 2))
    rest = g.choice([d for d in range(1, 16) if d != d0], size=half - 1, replace=False)
    digits = [int(d0)] + [int(x) for x in rest] + [int(x) for x in up]
    return sum(d << (4 * i) for i, d in enumerate(digits))


def _dev(keys):
    return torch.tensor(keys, dtype=torch.uint64).view(torch.int64).cuda() if False else \
        torch.from_numpy(np.array(keys, dtype=np.uint64).view(np.int64)).cuda()


@pytest.mark.parametrize("W", [8, 10, 16, 20, 24])
def test_small_widths_match_oracle(sq, W):
    g = np.random.Generator(np.random.PCG64(W))
    keys = [_scaled_key(g, max(W, 8)) & ((1 << W) - 1) | 1 for _ in range(3)] + [0, (1 << W) - 1]
    h = sq.scaled_hist(W, _dev(keys))
    torch.cuda.synchronize()
    got = h.cpu().numpy().view(np.uint64)
    for i, k in enumerate(keys):
        want = O.scaled_hist_range(k, W, 0, 1 << W)
        assert np.array_equal(got[i], want), (W, hex(k))


def test_w32_one_key_matches_parallel_oracle(sq):
    g = np.random.Generator(np.random.PCG64(32))
    key = _scaled_key(g, 32)
    h = sq.scaled_hist(32, _dev([key]))
    torch.cuda.synchronize()
    got = h.cpu().numpy().view(np.uint64)[0]
    parts = 64
    step = (1 << 32) // parts
    with ThreadPoolExecutor(ncores()) as ex:
        hs = list(ex.map(lambda i: O.scaled_hist_range(key, 32, i * step, step), range(parts)))
    want = np.sum(hs, axis=0, dtype=np.uint64)
    assert np.array_equal(got, want)


def test_w32_key_zero_single_bin(sq):
    h = sq.scaled_hist(32, _dev([0]))
    torch.cuda.synchronize()
    got = h.cpu().numpy().view(np.uint64)[0]
    assert got[0] == 1 << 32 and got[1:].sum() == 0


def test_w32_uniformity_claim(sq):
    import paper_2004_06278_b200.battery as B
    g = np.random.Generator(np.random.PCG64(2004))
    keys = [_scaled_key(g, 32) for _ in range(32)]
    res = B.scaled_uniformity(32, keys)
    assert sum(p > 1e-4 for _, p in res) >= 0.9 * len(keys), res
