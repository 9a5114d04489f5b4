"""Plain pinned D2H bandwidth (one 4 GiB copy): the PCIe ceiling the e2e number is held against."""
import torch, time
n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda"); h = torch.empty(n, dtype=torch.uint8).pin_memory()
for _ in range(2): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
print("D2H pinned 4 GiB: %.1f GB/s" % (n / best / 1e9))
