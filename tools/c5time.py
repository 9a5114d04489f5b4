"""Times the c5 kernel of the loaded library (SQ_LIB / SQ_FUSED_IMPL select the build): 2^34
samples per launch, best and median of R rounds of 5 launches; prints one JSON line."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import paper_2004_06278_b200 as sq  # noqa: E402

torch.cuda.set_device(0)
key = int(sq.keygen(1, 1)[0]) & ((1 << 64) - 1)
n = 1 << 34
h = torch.zeros(65536, dtype=torch.int64, device="cuda")
o = torch.zeros(32, dtype=torch.int64, device="cuda")
sq.fused_stats(key, 0, n, h, o)
torch.cuda.synchronize()
rates = []
for _ in range(int(os.environ.get("ROUNDS", "6"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sq.fused_stats(key, 0, n, h, o)
    e1.record()
    torch.cuda.synchronize()
    rates.append(5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print(json.dumps({"lib": os.environ.get("SQ_LIB", "product"), "impl": os.environ.get("SQ_FUSED_IMPL", "default"),
                  "tag": sys.argv[1] if len(sys.argv) > 1 else "", "best": max(rates),
                  "median": statistics.median(rates)}))
