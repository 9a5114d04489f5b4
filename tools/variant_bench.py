"""Times experimental builds of libsquares.so side by side on one GPU.

    python tools/variant_bench.py lib1.so lib2.so ...
Each library is loaded with ctypes (RTLD_LOCAL) and timed on c2 (fill_u32, 2^30), c3 (fill_u64,
2^29), c4 (fill_f32, 4096 x 2^18) and a 2^34-counter fused run; prints one JSON line per lib.
"""
import ctypes
import json
import sys

import torch


def load(path):
    L = ctypes.CDLL(path)
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    for f in ("sq_fill_u32", "sq_fill_u64", "sq_fill_f32"):
        getattr(L, f).argtypes = [vp, u64, u64, u64, vp, u64, vp]
    L.sq_fused_stats.argtypes = [u64, u64, u64, vp, vp, vp]
    for f in ("sq_fill_u32_k", "sq_fill_u64_k", "sq_fill_f32_k"):
        if hasattr(L, f):
            getattr(L, f).argtypes = [u64, u64, u64, vp, vp]
    return L


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    key = 0x1fac726d8cb5432f
    keys1 = torch.tensor([key], dtype=torch.int64, device="cuda")
    keys4096 = torch.randint(1, 1 << 62, (4096,), dtype=torch.int64, device="cuda") | 1
    out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    o = torch.zeros(32, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for path in sys.argv[1:]:
        L = load(path)
        r = {"lib": path}
        ms = timeit(lambda: L.sq_fill_u32(keys1.data_ptr(), 1, 0, 1 << 30, out.data_ptr(), 1 << 30, s), 30)
        r["c2_gsps"] = (1 << 30) / ms / 1e6
        if hasattr(L, "sq_fill_u32_k"):
            ms = timeit(lambda: L.sq_fill_u32_k(key, 0, 1 << 30, out.data_ptr(), s), 30)
            r["c2k_gsps"] = (1 << 30) / ms / 1e6
            ms = timeit(lambda: L.sq_fill_u64_k(key, 0, 1 << 29, out.data_ptr(), s), 30)
            r["c3k_gsps"] = (1 << 29) / ms / 1e6
        ms = timeit(lambda: L.sq_fill_u64(keys1.data_ptr(), 1, 0, 1 << 29, out.data_ptr(), 1 << 29, s), 30)
        r["c3_gsps"] = (1 << 29) / ms / 1e6
        ms = timeit(lambda: L.sq_fill_f32(keys4096.data_ptr(), 4096, 0, 1 << 18, out.data_ptr(), 1 << 18, s), 30)
        r["c4_gsps"] = (1 << 30) / ms / 1e6
        ms = timeit(lambda: L.sq_fused_stats(key, 0, 1 << 34, h.data_ptr(), o.data_ptr(), s), 3)
        r["c5_gsps"] = (1 << 34) / ms / 1e6
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
