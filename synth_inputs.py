"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no squaring, no key rules, no Weyl
stepping): only the workload shapes of BASELINE.json's configs, seeded uniform 64-bit
draws from numpy's PCG64 for fuzzing, and the edge-case lists of SURVEY.md §8(d).
Keys for the configs come from the key utility ("different digits"); the
caller decides which implementation (oracle or product) draws them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1

# Fuzz seed documented in SURVEY.md §8(d) ("seed 20040627").
FUZZ_SEED = 20040627


@dataclass(frozen=True)
class Workload:
    name: str          # c1..c5 (BASELINE.json configs[0..4])
    kind: str          # u32 | u64 | f32 | fused
    key_seed: int      # seed passed to the key utility
    nkeys: int         # keys drawn from that seed
    ctr0: int
    n: int             # counters per key
    shard: str         # "ctr" (counter-sharded) or "key" (key-sharded) across ranks

    @property
    def samples(self) -> int:
        return self.nkeys * self.n

    @property
    def elem_bytes(self) -> int:
        return {"u32": 4, "f32": 4, "u64": 8, "fused": 0}[self.kind]


# BASELINE.json "configs" (lines 7-11), in order.
CONFIGS = {
    "c1": Workload("c1", "u32", 1, 1, 0, 1 << 20, "ctr"),
    "c2": Workload("c2", "u32", 1, 1, 0, 1 << 30, "ctr"),
    "c3": Workload("c3", "u64", 1, 1, 0, 1 << 29, "ctr"),
    "c4": Workload("c4", "f32", 7, 4096, 0, 1 << 18, "key"),
    "c5": Workload("c5", "fused", 1, 1, 0, 1 << 38, "ctr"),
}

# Corner values for ctr and key (SURVEY.md §8(c) "corner set").
CORNERS = [0, 1, 2, 3, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 1 << 63, (1 << 63) + 1,
           M64 - 1, M64]


def random_pairs(n: int, seed: int = FUZZ_SEED):
    """n seeded uniform (ctr, key) pairs plus the full corner cross product, as uint64 arrays."""
    g = np.random.Generator(np.random.PCG64(seed))
    ctr = g.integers(0, 1 << 64, size=n, dtype=np.uint64, endpoint=False)
    key = g.integers(0, 1 << 64, size=n, dtype=np.uint64, endpoint=False)
    cc = np.array([a for a in CORNERS for _ in CORNERS], dtype=np.uint64)
    kk = np.array([b for _ in CORNERS for b in CORNERS], dtype=np.uint64)
    return np.concatenate([ctr, cc]), np.concatenate([key, kk])


def random_u64(n: int, seed: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(seed))
    return g.integers(0, 1 << 64, size=n, dtype=np.uint64, endpoint=False)


def sample_indices(n: int, count: int, seed: int, window: int = 4096) -> np.ndarray:
    """Sorted, unique indices into [0, n): `count` seeded uniform draws plus the first and
    last `window` indices (head and ragged tail of a full-size output)."""
    g = np.random.Generator(np.random.PCG64(seed))
    idx = g.integers(0, n, size=count, dtype=np.int64)
    head = np.arange(min(window, n), dtype=np.int64)
    tail = np.arange(max(0, n - window), n, dtype=np.int64)
    return np.unique(np.concatenate([idx, head, tail]))


# Fill edge cases (SURVEY.md §8(d) "Edge runs"): (ctr0, n, nkeys, ld_pad, out_offset_elems).
FILL_EDGES = [
    (0, 0, 1, 0, 0),                       # n = 0: no-op
    (0, 1, 1, 0, 0),
    (0, 3, 1, 0, 0),
    (0, 5, 1, 0, 0),
    (M64 - 4, 10, 1, 0, 0),                # counter wraps mod 2^64
    ((1 << 32) - 3, 1000, 1, 0, 0),        # 32-bit carry in ctr
    (12345, (1 << 20) + 3, 1, 0, 0),       # several tiles and a ragged tail
    (7, 777, 1, 0, 1),                     # output pointer offset by one element
    (0, 1000, 3, 7, 0),                    # nkeys = 3 with ld = n + 7 (sentinel padding)
    (99, 4099, 5, 1, 3),                   # ragged everything
]
