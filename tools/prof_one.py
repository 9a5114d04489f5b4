"""Run one config once (warm-up + 1 launch) from a given library: python exp/prof_one.py lib.so cfg"""
import ctypes, sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from variant_bench import load
L = load(sys.argv[1]); cfg = sys.argv[2]
key = 0x1fac726d8cb5432f
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
h = torch.zeros(65536, dtype=torch.int64, device="cuda"); o = torch.zeros(32, dtype=torch.int64, device="cuda")
keys4096 = torch.randint(1, 1 << 62, (4096,), dtype=torch.int64, device="cuda") | 1
f = {"c2": lambda: L.sq_fill_u32_k(key, 0, 1 << 30, out.data_ptr(), s),
     "c3": lambda: L.sq_fill_u64_k(key, 0, 1 << 29, out.data_ptr(), s),
     "c4": lambda: L.sq_fill_f32(keys4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s),
     "c5": lambda: L.sq_fused_stats(key, 0, 1 << 33, h.data_ptr(), o.data_ptr(), s)}[cfg]
for _ in range(2): f()
torch.cuda.synchronize()
