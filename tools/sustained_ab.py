"""Sustained (power-capped) A/B timing of library builds on one workload: warm the board into its
power-limited steady state, then alternate the libraries in blocks of launches.

    python tools/sustained_ab.py c2 lib1.so lib2.so ...
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from variant_bench import load  # noqa: E402

cfg = sys.argv[1]
libs = [(p, load(p)) for p in sys.argv[2:]]
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
h = torch.zeros(65536, dtype=torch.int64, device="cuda")
o = torch.zeros(32, dtype=torch.int64, device="cuda")
k4096 = torch.randint(1, 1 << 62, (4096,), dtype=torch.int64, device="cuda") | 1
key = 0x1fac726d8cb5432f


def step(L):
    if cfg == "c2":
        return L.sq_fill_u32_k(key, 0, 1 << 30, out.data_ptr(), s), 1 << 30
    if cfg == "c3":
        return L.sq_fill_u64_k(key, 0, 1 << 29, out.data_ptr(), s), 1 << 29
    if cfg == "c4":
        return L.sq_fill_f32(k4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s), 1 << 30
    return L.sq_fused_stats(key, 0, 1 << 32, h.data_ptr(), o.data_ptr(), s), 1 << 32


def block(L, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _, n = step(L)
    e1.record()
    torch.cuda.synchronize()
    return n / (e0.elapsed_time(e1) / reps) / 1e6


for _, L in libs:           # first launch of each library (module load) outside the timing
    block(L, 1)
for _ in range(8):          # ~5 s of load: into the power-capped steady state
    block(libs[0][1], 100)
res = {p: [] for p, _ in libs}
for rnd in range(6):
    for p, L in libs:
        res[p].append(block(L, 100))
for p, v in res.items():
    print(f"{p}: median {statistics.median(v):.1f} Gsamples/s  ({', '.join(f'{x:.0f}' for x in v)})")
