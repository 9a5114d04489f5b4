"""Launch-bound regime (BASELINE.json config 1 size and below): time per call of sq_fill_u32_k
issued eagerly vs replayed from a CUDA graph of 64 calls.  python tools/small_n.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_06278_b200 as sq  # noqa: E402

key = int(sq.keygen(1, 1)[0]) & ((1 << 64) - 1)
s = torch.cuda.Stream()
for n in (1 << 12, 1 << 16, 1 << 20):
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(10):
            sq.fill_u32_k(key, 0, n, out=out, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for i in range(640):
            sq.fill_u32_k(key, i * n, n, out=out, stream=s)
        e1.record(s)
    torch.cuda.synchronize()
    eager_us = e0.elapsed_time(e1) * 1e3 / 640
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(64):
            sq.fill_u32_k(key, i * n, n, out=out, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) * 1e3 / 640
    print(f"n = 2^{n.bit_length() - 1}: eager {eager_us:7.2f} us/call ({n / eager_us / 1e3:7.1f} Gsamples/s), "
          f"graph {graph_us:7.2f} us/call ({n / graph_us / 1e3:7.1f} Gsamples/s)")
