"""Test helpers: run the (single-threaded) oracle over disjoint shards on all host cores.

ctypes releases the GIL during foreign calls, so a thread pool runs one oracle loop per core.
Nothing here does the method's arithmetic; it only splits ranges and concatenates results.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle as O


def ncores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _splits(n: int, parts: int):
    q, r = divmod(n, parts)
    s = 0
    for i in range(parts):
        ln = q + (1 if i < r else 0)
        yield s, ln
        s += ln


def par_fill(kind: str, key: int, ctr0: int, n: int, threads: int | None = None) -> np.ndarray:
    """oracle.fill(kind, [key], ctr0, n)[0] computed as `threads` contiguous shards."""
    threads = threads or ncores()
    parts = [(s, ln) for s, ln in _splits(n, max(1, min(threads * 4, n))) if ln]
    with ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda p: O.fill(kind, [key], ctr0 + p[0], p[1])[0], parts))
    return np.concatenate(outs) if outs else np.zeros(0)


def par_fused(key: int, ctr0: int, n: int, threads: int | None = None):
    threads = threads or ncores()
    parts = [(s, ln) for s, ln in _splits(n, max(1, min(threads * 4, n))) if ln]
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(lambda p: O.fused_stats(key, ctr0 + p[0], p[1]), parts))
    h = np.zeros(65536, np.uint64)
    o = np.zeros(32, np.uint64)
    for hh, oo in res:
        h += hh
        o += oo
    return h, o


def first_mismatch(got: np.ndarray, want: np.ndarray) -> str:
    bad = np.nonzero(got != want)[0]
    if bad.size == 0:
        return "no mismatch"
    i = int(bad[0])
    return f"{bad.size} mismatches; first at {i}: got {got[i]!r} want {want[i]!r}"
