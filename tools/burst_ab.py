"""Burst A/B timing of library builds on the store-bound configs: each measurement is 5
launches after a 0.5 s idle gap (so the board's power limit, which a sustained 4 GiB fill
reaches after a few hundred launches, does not decide the comparison); libraries alternate,
R rounds, median per (lib, config).  python tools/burst_ab.py lib1.so lib2.so ..."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from variant_bench import load  # noqa: E402

key = 0x1fac726d8cb5432f
keys1 = torch.tensor([key], dtype=torch.int64, device="cuda")
g = torch.Generator().manual_seed(7)
keys4096 = (torch.randint(1, 1 << 62, (4096,), dtype=torch.int64, generator=g) | 1).cuda()
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
libs = [(p, load(p)) for p in sys.argv[1:]]
cfgs = {
    "c2k": (1 << 30, lambda L: L.sq_fill_u32_k(key, 0, 1 << 30, out.data_ptr(), s)),
    "c2dev": (1 << 30, lambda L: L.sq_fill_u32(keys1.data_ptr(), 1, 0, 1 << 30, out.data_ptr(), 1 << 30, s)),
    "c3k": (1 << 29, lambda L: L.sq_fill_u64_k(key, 0, 1 << 29, out.data_ptr(), s)),
    "c4": (1 << 30, lambda L: L.sq_fill_f32(keys4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s)),
}
res = {(p, c): [] for p, _ in libs for c in cfgs}
for _ in range(int(__import__("os").environ.get("ROUNDS", "5"))):
    for c, (n, f) in cfgs.items():
        for p, L in libs:
            torch.cuda.synchronize()
            time.sleep(0.5)
            f(L)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                f(L)
            e1.record()
            torch.cuda.synchronize()
            res[(p, c)].append(5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
for p, _ in libs:
    print(json.dumps({"lib": p, **{c: round(statistics.median(res[(p, c)]), 1) for c in cfgs}}))
