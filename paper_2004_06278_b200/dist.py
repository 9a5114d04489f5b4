"""Multi-GPU composition: counter- or key-sharding, one process per GPU.

PAPER.md P:41: "If the 2^64 is divided equally among all the cores, one could provide a stream
of about 1.8 trillion random numbers per core."  Every output is a pure function of
(ctr, key) ("there is no state"), so the fills shard with NO data-path collective: each
rank writes its own contiguous counter range (or its own key rows) into its own HBM.  The fused
statistics have one real exchange step: an all-reduce SUM of the 65,536 + 32 counts.

The host logic here (partition, packing, the all-reduce) is device-agnostic: the CPU tests run
it over the gloo backend with world_size 2; on GPUs it runs over NCCL.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as tdist

HIST_BINS = 65536


def partition(n: int, parts: int, idx: int) -> tuple[int, int]:
    """(start, length) of part `idx` when [0, n) is divided into `parts` contiguous pieces:
    floor(n / parts) each, the last absorbing the remainder.  n may be 2^64
    (a shard of length 2^64 cannot be passed to the C ABI in one call: the bindings reject it)."""
    if parts < 1 or not (0 <= idx < parts):
        raise ValueError("need parts >= 1 and 0 <= idx < parts")
    q = n // parts
    start = idx * q
    return start, (n - start) if idx == parts - 1 else q


def rank_world(group=None) -> tuple[int, int]:
    if tdist.is_available() and tdist.is_initialized():
        return tdist.get_rank(group), tdist.get_world_size(group)
    return 0, 1


def counter_shard(ctr0: int, n: int, group=None) -> tuple[int, int]:
    """This rank's (first counter, count) of [ctr0, ctr0 + n) (counters wrap mod 2^64)."""
    r, p = rank_world(group)
    s, ln = partition(n, p, r)
    return (ctr0 + s) & ((1 << 64) - 1), ln


def key_shard(nkeys: int, group=None) -> tuple[int, int]:
    """This rank's (first key row, row count) of nkeys rows (BASELINE.json config 4)."""
    r, p = rank_world(group)
    return partition(nkeys, p, r)


def counts_buffer(device=None) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """One zeroed packed int64 buffer of 65,568 counts and its two views (hist = the first
    65,536, ones = the last 32), so the exchange below runs in place on a single tensor."""
    buf = torch.zeros(HIST_BINS + 32, dtype=torch.int64, device=device)
    return buf, buf[:HIST_BINS], buf[HIST_BINS:]


def _packed(hist: torch.Tensor, ones: torch.Tensor) -> torch.Tensor | None:
    """The packed buffer hist and ones are views of (counts_buffer), else None."""
    if not (hist.is_contiguous() and ones.is_contiguous() and hist.numel() == HIST_BINS and ones.numel() == 32):
        return None
    if hist.untyped_storage().data_ptr() != ones.untyped_storage().data_ptr():
        return None
    if ones.data_ptr() != hist.data_ptr() + HIST_BINS * hist.element_size():
        return None
    return hist.view(-1).as_strided((HIST_BINS + 32,), (1,))


def allreduce_counts(hist: torch.Tensor, ones: torch.Tensor, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """SUM-all-reduce hist (65536) and ones (32) int64 counts in ONE collective over one packed
    65,568-element buffer (524,544 bytes): in place when hist and ones are the two views of
    counts_buffer(), else through a packed copy.  Integer addition is associative and
    commutative, so the result is bit-identical for any world size and rank order."""
    if not (tdist.is_available() and tdist.is_initialized()):
        return hist, ones
    buf = _packed(hist, ones)
    if buf is not None:
        tdist.all_reduce(buf, op=tdist.ReduceOp.SUM, group=group)
        return hist, ones
    buf = torch.cat([hist.reshape(-1), ones.reshape(-1)])
    tdist.all_reduce(buf, op=tdist.ReduceOp.SUM, group=group)
    hist.copy_(buf[:HIST_BINS])
    ones.copy_(buf[HIST_BINS:])
    return hist, ones


def fused_stats_sharded(key: int, ctr0: int, n: int,
                        local: Callable[[int, int, int], tuple[torch.Tensor, torch.Tensor]] | None = None,
                        group=None, device=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Counter-sharded fused statistics: rank r computes its shard with `local(key, c0, ln)`
    (default: the CUDA kernel, paper_2004_06278_b200.fused_stats, accumulating into one packed
    counts buffer on `device`), then one in-place all-reduce."""
    if local is None:
        from . import fused_stats as _fused

        def local(k, c0, ln):
            _, h, o = counts_buffer(device if device is not None else "cuda")
            return _fused(k, c0, ln, hist=h, ones=o)
    c0, ln = counter_shard(ctr0, n, group)
    hist, ones = local(key, c0, ln)
    return allreduce_counts(hist, ones, group)
