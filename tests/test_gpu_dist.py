"""GPU tests (-m gpu) of the sharded path with the REAL kernels: P
processes, each running the CUDA kernels on its own shard, then the one exchange step.

PAPER.md P:41: the counter space "divided equally among all the cores".  Every process runs on
cuda:0 (the box has one GPU) and the process group is gloo over CUDA tensors (NCCL refuses two
ranks on one device); the per-rank code is the product's multi-GPU code path verbatim
(paper_2004_06278_b200.dist: partition, fused_stats_sharded with the default CUDA kernel, the
in-place all-reduce of the packed counts buffer).  Nothing waits on another rank's kernel: each
rank's kernels finish before the collective, so the ranks sharing one GPU never deadlock.
Results are compared with the single-process oracle element by element / count by count.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, job, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2004_06278_b200 as sq
        from paper_2004_06278_b200 import dist as D
        kind = job["kind"]
        if kind == "fused":
            hist, ones = D.fused_stats_sharded(job["key"], job["ctr0"], job["n"], device="cuda:0")
            torch.cuda.synchronize()
            q.put((rank, "fused", hist.cpu().numpy().view(np.uint64).copy(), ones.cpu().numpy().view(np.uint64).copy(),
                   D.counter_shard(job["ctr0"], job["n"])))
        elif kind == "keyshard_f32":
            # BASELINE.json config 4's layout: rank r fills its own block of key rows
            keys = torch.tensor(np.asarray(job["keys"], dtype=np.uint64).view(np.int64))
            k0, kn = D.key_shard(keys.numel())
            out = sq.fill_f32(keys[k0:k0 + kn].cuda(), job["ctr0"], job["n"])
            torch.cuda.synchronize()
            q.put((rank, kind, out.cpu().numpy().view(np.uint32).copy(), None, (k0, kn)))
        elif kind == "ctrshard_u32":
            # BASELINE.json config 2's layout: rank r fills its own contiguous counter block
            c0, ln = D.counter_shard(job["ctr0"], job["n"])
            out = sq.fill_u32_k(job["key"], c0, ln, device="cuda:0")
            torch.cuda.synchronize()
            q.put((rank, kind, out.cpu().numpy().view(np.uint32).copy(), None, (c0, ln)))
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def _run(world, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world", [2, 3])
def test_fused_sharded_cuda_kernel_allreduce(world):
    """a1 + a7 + a8: each rank runs the fused CUDA kernel on its counter shard of a range that
    straddles the 2^64 wrap (ragged: n = 2^24 + 7), then the one in-place all-reduce; every rank
    holds the full-range counts, equal to the single-process oracle."""
    key = int(O.keygen(1, 1)[0])
    ctr0, n = (1 << 64) - (1 << 20), (1 << 24) + 7
    res = _run(world, {"kind": "fused", "key": key, "ctr0": ctr0, "n": n})
    hw, ow = O.fused_stats(key, ctr0, n)
    pos = ctr0
    for _, _, h, o, (c0, ln) in res:
        assert np.array_equal(h, hw) and np.array_equal(o, ow)
        assert c0 == pos & M64
        pos += ln
    assert pos - ctr0 == n


@pytest.mark.parametrize("world", [2, 3])
def test_key_sharded_f32_fill(world):
    """BASELINE.json config 4 shape (keys from seed 7, [key][ctr] float32) sharded by key rows:
    the rows of all ranks, concatenated in rank order, equal the oracle's fill bit for bit."""
    keys = O.keygen(7, 67)                      # ragged: 67 rows over 2 or 3 ranks
    ctr0, n = 0, (1 << 14) + 3
    res = _run(world, {"kind": "keyshard_f32", "keys": keys.tolist(), "ctr0": ctr0, "n": n})
    got = np.concatenate([r[2] for r in res], axis=0)
    want = O.fill("f32", keys, ctr0, n).view(np.uint32)
    assert got.shape == want.shape and np.array_equal(got, want)
    assert [r[4][0] for r in res] == [sum(x[4][1] for x in res[:i]) for i in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_counter_sharded_u32_fill(world):
    """BASELINE.json config 2 shape (one key, seed 1) sharded by counter blocks through the
    key-by-value entry point the bench times; the blocks concatenated equal the oracle."""
    key = int(O.keygen(1, 1)[0])
    ctr0, n = (1 << 32) - 1000, (1 << 22) + 5
    res = _run(world, {"kind": "ctrshard_u32", "key": key, "ctr0": ctr0, "n": n})
    got = np.concatenate([r[2] for r in res])
    want = O.fill("u32", [key], ctr0, n)[0]
    assert np.array_equal(got, want)
