"""A/B c5 timing: alternate libraries, several rounds; python exp/c5ab.py lib1 lib2 ..."""
import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from variant_bench import load, timeit
libs = [(p, load(p)) for p in sys.argv[1:]]
key = 0x1fac726d8cb5432f
h = torch.zeros(65536, dtype=torch.int64, device="cuda"); o = torch.zeros(32, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
res = {p: [] for p, _ in libs}
for rnd in range(4):
    for p, L in libs:
        ms = timeit(lambda: L.sq_fused_stats(key, 0, 1 << 34, h.data_ptr(), o.data_ptr(), s), 5)
        res[p].append(round((1 << 34) / ms / 1e6, 1))
for p, v in res.items():
    print(p, v, "best", max(v))
