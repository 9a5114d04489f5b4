"""Measurement of the SURVEY 8(f) ("next") rows on one GPU, each against its roofline:
python tools/bench_next.py > profiles/r01_bench_next.jsonl

Fills and key-counter mode: algorithmic HBM bytes / time vs the measured copy peak
(MEASURED_PEAKS.json).  Statistics and the device API: samples / time vs the 9-slot multiply
floor of squares32 (64/9 samples/clk/SM x SMs x max clock), the same roofline bench.py uses for
c5.  Best of 5 timed launches after a warm-up, CUDA events on the launching stream."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_06278_b200 as sq  # noqa: E402
from paper_2004_06278_b200 import _build  # noqa: E402


def best_ms(fn, reps=5):
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


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    floor = 64.0 / 9.0 * sms * mhz * 1e6 / 1e9   # Gsamples/s
    key = int(sq.keygen(1, 1)[0]) & ((1 << 64) - 1)
    out = torch.empty(1 << 32, dtype=torch.uint8, device="cuda")   # 4 GiB scratch
    rows = []

    def fill_row(name, n, bytes_per, fn):
        ms = best_ms(fn)
        gbs = n * bytes_per / (ms * 1e-3) / 1e9
        rows.append({"row": name, "samples": n, "ms": ms, "Gsamples_per_s": n / (ms * 1e-3) / 1e9,
                     "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                  "algorithmic_bytes_per_sample": bytes_per}})

    def alu_row(name, n, fn, slots=9):
        ms = best_ms(fn)
        g = n / (ms * 1e-3) / 1e9
        pk = floor * 9.0 / slots
        rows.append({"row": name, "samples": n, "ms": ms, "Gsamples_per_s": g,
                     "roofline": {"bound": "alu", "achieved": g, "peak": pk, "unit": "Gsamples/s",
                                  "frac": g / pk, "peak_note": f"{slots}-slot multiply floor"}})

    n29, n30 = 1 << 29, 1 << 30
    f64 = out.view(torch.float64)[:n29]
    fill_row("8(f)1 squares64 -> f64 fill, 2^29, key by value", n29, 8, lambda: sq.fill_f64_k(key, 0, n29, out=f64))
    f2 = out.view(torch.float32)[:2 * n29].view(n29, 2)
    fill_row("8(f)1 squares64 -> 2 x f32 fill, 2^29, key by value", n29, 8,
             lambda: sq.fill_f32x2_k(key, 0, n29, out=f2))
    u32 = out.view(torch.int32)[:n30]
    fill_row("8(f)2 strided u32 fill (stride 3), 2^30", n30, 4,
             lambda: sq.fill_ex("u32", 0, n30, stride=3, key=key, out=u32))
    nk = 1 << 28
    keys = torch.randint(1, 1 << 62, (nk,), dtype=torch.int64, device="cuda") | 1
    k32 = out.view(torch.int32)[:nk]
    fill_row("8(f)2 key-counter mode u32, 2^28 keys (8 B read + 4 B written)", nk, 12,
             lambda: sq.fill_keyctr("u32", keys, 12345, out=k32))
    del keys
    h = torch.zeros(65536, dtype=torch.int64, device="cuda")
    o = torch.zeros(32, dtype=torch.int64, device="cuda")
    n34 = 1 << 34
    alu_row("8(f)2 fused statistics, bit-reversed, stride 3, 2^34", n34,
            lambda: sq.fused_stats_ex(key, 0, n34, stride=3, bitrev=True, hist=h, ones=o))
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    alu_row("8(f)3 transitions (runs), 2^34", n34, lambda: sq.transitions(key, 0, n34, count=c))
    kk = torch.randint(1, 1 << 62, (8,), dtype=torch.int64, device="cuda") | 1
    hs = torch.zeros((8, 65536), dtype=torch.int64, device="cuda")
    alu_row("8(f)3 exhaustive W = 32 histograms, 8 keys x 2^32 (32-bit arithmetic: 4 IMAD/sample)", 8 << 32,
            lambda: sq.scaled_hist(32, kk, hist=hs), slots=4)
    lib = ctypes.CDLL(_build.build_devapi_test())
    lib.devapi_stream_xor.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_void_p]
    blocks, per = sms * 8, 1 << 12
    acc = torch.empty(blocks * 256, dtype=torch.int32, device="cuda")
    alu_row(f"8(f)4 device API sq::Stream::next_u32, XOR-folded ({blocks * 256} threads x {per})",
            blocks * 256 * per, lambda: lib.devapi_stream_xor(key, 0, per, blocks, acc.data_ptr()))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
