"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic in
paper_2004_06278_b200/dist.py: partition rule, counter/key shards, and the single all-reduce of
the fused counts.  The per-shard compute is injected (here: the CPU oracle standing in for the
CUDA kernel, which needs a GPU); what is under test is the sharding and the exchange step.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, key, ctr0, n, nkeys, q, perm=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2004_06278_b200 import dist as D

        def local(k, c0, ln):
            h, o = O.fused_stats(k, c0, ln)
            if rank % 2:   # odd ranks: separate tensors (the packed-copy path of allreduce_counts)
                return torch.from_numpy(h.view(np.int64).copy()), torch.from_numpy(o.view(np.int64).copy())
            _, hv, ov = D.counts_buffer()   # even ranks: views of one buffer (the in-place path)
            hv.copy_(torch.from_numpy(h.view(np.int64)))
            ov.copy_(torch.from_numpy(o.view(np.int64)))
            return hv, ov

        if perm is None:
            hist, ones = D.fused_stats_sharded(key, ctr0, n, local=local)
        else:   # permuted rank -> shard map: rank r computes shard perm[r], then the one all-reduce
            s0, sl = D.partition(n, world, perm[rank])
            hist, ones = D.allreduce_counts(*local(key, (ctr0 + s0) & ((1 << 64) - 1), sl))
        c0, ln = D.counter_shard(ctr0, n)
        k0, kn = D.key_shard(nkeys)
        # every rank gets the same reduced counts; report the shard geometry too
        q.put((rank, hist.numpy().view(np.uint64).copy(), ones.numpy().view(np.uint64).copy(), (c0, ln), (k0, kn)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,perm", [(2, None), (3, None), (4, None), (8, None), (4, (2, 0, 3, 1))])
def test_fused_sharded_allreduce_matches_single(world, perm):
    """P = 2, 3, 4, 8 ranks (and a permuted rank -> shard map): the all-reduced counts equal the
    single-process oracle bit for bit, and the shards tile the counter range."""
    key = int(O.keygen(1, 1)[0])
    ctr0, n, nkeys = (1 << 64) - 50_000, 300_001, 10   # shards straddle the 2^64 wrap; ragged
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, key, ctr0, n, nkeys, q, perm)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    h_want, o_want = O.fused_stats(key, ctr0, n)
    for _, h, o, _, _ in res:
        assert np.array_equal(h, h_want) and np.array_equal(o, o_want)
    # shards are contiguous, disjoint, cover [ctr0, ctr0+n) (mod 2^64); key shards cover nkeys
    pos = ctr0
    total = 0
    kpos = 0
    for r, _, _, (c0, ln), (k0, kn) in res:
        assert c0 == pos & ((1 << 64) - 1)
        pos += ln
        total += ln
        assert k0 == kpos
        kpos += kn
    assert total == n and kpos == nkeys


def test_partition_matches_oracle_rule():
    from paper_2004_06278_b200 import dist as D
    for n in [0, 1, 5, 1 << 30, (1 << 38) + 7, 1 << 64]:
        for parts in [1, 2, 3, 4, 8, 7]:
            for i in range(parts):
                assert D.partition(n, parts, i) == O.partition(n, parts, i)
    with pytest.raises(ValueError):
        D.partition(10, 0, 0)


def test_allreduce_without_process_group_is_identity():
    from paper_2004_06278_b200 import dist as D
    h = torch.arange(65536, dtype=torch.int64)
    o = torch.arange(32, dtype=torch.int64)
    h2, o2 = D.allreduce_counts(h.clone(), o.clone())
    assert torch.equal(h, h2) and torch.equal(o, o2)


def test_counts_buffer_views():
    """hist / ones from counts_buffer are recognised as one packed buffer (in-place exchange);
    separate tensors or other views are not."""
    from paper_2004_06278_b200 import dist as D
    buf, h, o = D.counts_buffer()
    assert buf.numel() == 65568 and h.numel() == 65536 and o.numel() == 32
    p = D._packed(h, o)
    assert p is not None and p.data_ptr() == buf.data_ptr() and p.numel() == 65568
    assert D._packed(h, torch.zeros(32, dtype=torch.int64)) is None
    assert D._packed(o, h) is None
