"""Separates the c4 costs: f32 vs u32 kind, 1 device key vs 4096 keys (same 2^30 samples)."""
import sys, torch, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from variant_bench import load, timeit
L = load(sys.argv[1] if len(sys.argv) > 1 else "paper_2004_06278_b200/libsquares.so")
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
k1 = torch.tensor([0x1fac726d8cb5432f], dtype=torch.int64, device="cuda")
k4096 = torch.randint(1, 1 << 62, (4096,), dtype=torch.int64, device="cuda") | 1
for name, f in [("u32 1 key", lambda: L.sq_fill_u32(k1.data_ptr(), 1, 0, 1 << 30, out.data_ptr(), 1 << 30, s)),
                ("f32 1 key", lambda: L.sq_fill_f32(k1.data_ptr(), 1, 0, 1 << 30, out.data_ptr(), 1 << 30, s)),
                ("u32 4096 keys", lambda: L.sq_fill_u32(k4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s)),
                ("f32 4096 keys", lambda: L.sq_fill_f32(k4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s)),
                ("f32_k 1 key", lambda: L.sq_fill_f32_k(0x1fac726d8cb5432f, 0, 1 << 30, out.data_ptr(), s))]:
    ms = timeit(f, 20)
    print(f"{name:16s} {(1 << 30) / ms / 1e6:8.1f} Gsamples/s")
