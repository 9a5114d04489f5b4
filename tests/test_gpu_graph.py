"""The C ABI's device entry points are CUDA-graph safe (-m gpu): they only enqueue work on the
caller's stream (no synchronisation, no allocation), so a user can capture a batch of small
fills and fused-statistics calls once and replay it -- the launch-bound small-n regime (config 1
size, 2^20 samples) -- with results identical to the oracle on every replay."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sq():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2004_06278_b200 as sq
    torch.cuda.set_device(0)
    return sq


def test_capture_and_replay(sq):
    key = int(O.keygen(1, 1)[0])
    keys = torch.from_numpy(O.keygen(7, 4).view(np.int64)).cuda()
    n = 1 << 20
    out_u = torch.empty(n, dtype=torch.int32, device="cuda")
    out_f = torch.empty((4, 4096), dtype=torch.float32, device="cuda")
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    ones = torch.zeros(32, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    # warm-up outside capture (first-launch attributes)
    with torch.cuda.stream(s):
        sq.fill_u32_k(key, 0, n, out=out_u, stream=s)
        sq.fill_f32(keys, 5, 4096, out=out_f, stream=s)
        sq.fused_stats(key, 0, n, hist, ones, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sq.fill_u32_k(key, 123, n, out=out_u, stream=s)
        sq.fill_f32(keys, 5, 4096, out=out_f, stream=s)
        hist.zero_()
        ones.zero_()
        sq.fused_stats(key, 77, n, hist, ones, stream=s)
    want_u = O.fill("u32", [key], 123, n)[0].view(np.uint32)
    want_f = O.fill("f32", O.keygen(7, 4), 5, 4096).view(np.uint32)
    want_h, want_o = O.fused_stats(key, 77, n)
    for _ in range(3):
        out_u.fill_(0)
        out_f.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out_u.cpu().numpy().view(np.uint32), want_u)
        assert np.array_equal(out_f.cpu().numpy().view(np.uint32), want_f)
        assert np.array_equal(hist.cpu().numpy().view(np.uint64), want_h)
        assert np.array_equal(ones.cpu().numpy().view(np.uint64), want_o)


def test_concurrent_host_threads_and_streams(sq):
    """Reentrancy (include/squares.h): 4 host threads, each with its own CUDA stream, issue fills
    and fused statistics concurrently (first-call caches included: a fresh process path is not
    needed, the caches are per device and atomic); every result equals the oracle."""
    import threading
    n = (1 << 18) + 3
    keys = [int(k) for k in O.keygen(21, 4)]
    results, errors = {}, []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs = []
                for rep in range(5):
                    kind = ("u32", "u64", "f32")[(t + rep) % 3]
                    outs.append((kind, rep, getattr(sq, f"fill_{kind}_k")(keys[t], rep * n, n, stream=s)))
                h, o = sq.fused_stats(keys[t], 7, n, stream=s)
            s.synchronize()
            results[t] = (outs, h.cpu().numpy().view(np.uint64), o.cpu().numpy().view(np.uint64))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors
    for t in range(4):
        outs, h, o = results[t]
        for kind, rep, out in outs:
            want = O.fill(kind, [keys[t]], rep * n, n)[0]
            got = out.cpu().numpy().view(want.dtype)
            assert np.array_equal(got, want), (t, kind, rep)
        hw, ow = O.fused_stats(keys[t], 7, n)
        assert np.array_equal(h, hw) and np.array_equal(o, ow), t
