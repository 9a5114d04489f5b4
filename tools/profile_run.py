"""Minimal launcher for ncu / compute-sanitizer: runs `reps` launches of one workload.

    python tools/profile_run.py --workload c2 --reps 3 [--n N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_06278_b200 as sq  # noqa: E402
import synth_inputs as SI  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0, help="override counters per key")
    a = ap.parse_args()
    w = SI.CONFIGS[a.workload]
    n = a.n or w.n
    keys = sq.keygen(w.key_seed, w.nkeys).cuda()
    if w.kind == "fused":
        h = torch.zeros(65536, dtype=torch.int64, device="cuda")
        o = torch.zeros(32, dtype=torch.int64, device="cuda")
        for _ in range(a.reps):
            sq.fused_stats(int(keys[0]), w.ctr0, n, h, o)
    else:
        dt = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32}[w.kind]
        out = torch.empty((w.nkeys, n), dtype=dt, device="cuda")
        for _ in range(a.reps):
            if w.nkeys == 1:   # same entry point as bench.py: key by value
                getattr(sq, f"fill_{w.kind}_k")(int(keys[0]), w.ctr0, n, out=out.view(-1))
            else:
                getattr(sq, f"fill_{w.kind}")(keys, w.ctr0, n, out=out)
    torch.cuda.synchronize()
    print("ok", a.workload, n)


if __name__ == "__main__":
    main()
