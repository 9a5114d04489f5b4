"""Context only ("faster than Philox"): bulk random fills of 2^30 32-bit
values on the same GPU with PyTorch's CUDA generator (Philox4x32-10) beside this repository's
squares32 fills.  Not a target; prints one JSON line per row."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_06278_b200 as sq  # noqa: E402


def best_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


n = 1 << 30
key = int(sq.keygen(1, 1)[0]) & ((1 << 64) - 1)
i32 = torch.empty(n, dtype=torch.int32, device="cuda")
f32 = torch.empty(n, dtype=torch.float32, device="cuda")
rows = [
    ("torch Philox4x32-10 int32 random_()", lambda: i32.random_()),
    ("torch Philox4x32-10 float32 uniform_()", lambda: f32.uniform_()),
    ("squares32 u32 fill (sq_fill_u32_k)", lambda: sq.fill_u32_k(key, 0, n, out=i32)),
    ("squares32 f32 fill (sq_fill_f32_k)", lambda: sq.fill_f32_k(key, 0, n, out=f32)),
]
for name, fn in rows:
    ms = best_ms(fn)
    print(json.dumps({"row": name, "samples": n, "ms": ms, "Gsamples_per_s": n / (ms * 1e-3) / 1e9,
                      "GBps": 4 * n / (ms * 1e-3) / 1e9}))
