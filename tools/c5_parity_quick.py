"""Quick c5-kernel parity for experimental builds (SQ_LIB=<lib> SQ_FUSED_IMPL=...): fused counts
vs the oracle on ragged sizes, hot bins (key 2^32), key 0 sweeps and the strided/bit-reversed
variants.  Exit code 1 on any mismatch."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import oracle as O  # noqa: E402
import paper_2004_06278_b200 as sq  # noqa: E402
from tests.helpers import par_fused  # noqa: E402

torch.cuda.set_device(0)
key = int(O.keygen(1, 1)[0])
bad = 0
cases = [(key, 77, n) for n in (1, 31, 33, 1000, 32768 * 3 + 7, (1 << 20) + 5, 1 << 22, (1 << 26) + 12345)]
cases += [(1 << 32, 0, 1 << 23), ((1 << 32) + (1 << 16), 3, (1 << 23) + 12345), (key, (1 << 64) - 5000, 1 << 24)]
for k, c0, n in cases:
    h, o = sq.fused_stats(k, c0, n)
    torch.cuda.synchronize()
    hw, ow = par_fused(k, c0, n) if n > (1 << 22) else O.fused_stats(k, c0, n)
    ok = np.array_equal(h.cpu().numpy().view(np.uint64), hw) and np.array_equal(o.cpu().numpy().view(np.uint64), ow)
    bad += not ok
    print(("ok  " if ok else "BAD ") + f"key={k:#x} ctr0={c0} n={n}", flush=True)
h, o = sq.fused_stats(0, 5, 1 << 30)
torch.cuda.synchronize()
ok = int(h[0]) == 1 << 30 and int(h[1:].sum()) == 0 and int(o.sum()) == 0
bad += not ok
print(("ok  " if ok else "BAD ") + "key=0 n=2^30 closed form")
for stride, rev in ((3, False), (1, True), (5, True)):
    h, o = sq.fused_stats_ex(key, 11, (1 << 20) + 3, stride=stride, bitrev=rev)
    torch.cuda.synchronize()
    hw, ow = O.fused_stats_ex(key, 11, stride, (1 << 20) + 3, rev)
    ok = np.array_equal(h.cpu().numpy().view(np.uint64), hw) and np.array_equal(o.cpu().numpy().view(np.uint64), ow)
    bad += not ok
    print(("ok  " if ok else "BAD ") + f"stride={stride} bitrev={rev}")
sys.exit(1 if bad else 0)
