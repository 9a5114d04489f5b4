"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / initcheck).
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Exits non-zero on a parity mismatch; sanitizer findings are reported by the tool itself."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2004_06278_b200 as sq  # noqa: E402


def main():
    torch.cuda.set_device(0)
    keys_np = O.keygen(1, 3)
    keys = torch.from_numpy(keys_np.view(np.int64)).cuda()
    n = 5000
    for kind in ("u32", "u64", "f32", "f64", "f32x2"):
        # misaligned-by-one output, padded rows, counter wrap
        es = 8 if kind in ("u64", "f64", "f32x2") else 4
        out = getattr(sq, f"fill_{kind}")(keys, (1 << 64) - 777, n, ld=n + 3)
        one = getattr(sq, f"fill_{kind}_k")(int(keys_np[0]), 5, 1001)
        ex = sq.fill_ex(kind, 9, 777, stride=3, keys=keys)
        kc = sq.fill_keyctr(kind, keys, 42)
    torch.cuda.synchronize()
    h, o = sq.fused_stats(int(keys_np[0]), 0, (1 << 21) + 5)
    h2, o2 = sq.fused_stats_ex(int(keys_np[0]), 0, 100_003, stride=7, bitrev=True)
    h3, o3 = sq.fused_stats(0, 0, 1 << 17)          # guard-bit fix-up path (single bin)
    t = sq.transitions(int(keys_np[0]), 0, 100_000)
    sh = sq.scaled_hist(16, keys)
    sh32 = sq.scaled_hist(20, keys[:1])
    torch.cuda.synchronize()
    hw, ow = O.fused_stats(int(keys_np[0]), 0, (1 << 21) + 5)
    ok = np.array_equal(h.cpu().numpy().view(np.uint64), hw) and np.array_equal(o.cpu().numpy().view(np.uint64), ow)
    ok &= int(h3[0].item()) == (1 << 17)
    print("sanitize_run parity:", "ok" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
