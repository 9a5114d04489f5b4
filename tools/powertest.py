import sys, time, threading, torch, pynvml
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__))); sys.path.insert(0, ".")
from variant_bench import load
L = load(sys.argv[1] if len(sys.argv) > 1 else "paper_2004_06278_b200/libsquares.so")
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")
h = torch.zeros(65536, dtype=torch.int64, device="cuda"); o = torch.zeros(32, dtype=torch.int64, device="cuda")
key = 0x1fac726d8cb5432f
f = {"c2": (lambda: L.sq_fill_u32_k(key, 0, 1 << 30, out.data_ptr(), s), 1 << 30),
     "c3": (lambda: L.sq_fill_u64_k(key, 0, 1 << 29, out.data_ptr(), s), 1 << 29),
     "c5": (lambda: L.sq_fused_stats(key, 0, 1 << 32, h.data_ptr(), o.data_ptr(), s), 1 << 32)}[cfg]
pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []; stop = threading.Event()
def mon():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000, pynvml.nvmlDeviceGetTemperature(hd, 0),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd)))
        time.sleep(0.01)
th = threading.Thread(target=mon); th.start()
evs = []
for blk in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): f[0]()
    e1.record(); torch.cuda.synchronize()
    t = time.time()
    ms = e0.elapsed_time(e1) / 100
    win = [x for x in samples if x[0] > t - 0.15]
    sm = sorted(x[1] for x in win); pw = [x[2] for x in win]; rs = set(); [rs.add(x[4]) for x in win]
    print(f"block {blk}: {f[1] / ms / 1e6:7.1f} Gs/s  sm_mhz med {sm[len(sm)//2] if sm else None} min {sm[0] if sm else None}  power max {max(pw) if pw else 0:.0f} W  temp {win[-1][3] if win else None}  reasons {sorted(hex(r) for r in rs)}", flush=True)
stop.set(); th.join()
