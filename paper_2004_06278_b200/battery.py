"""GPU-resident desk battery ("a basic uniformity test",
"bits-reversed tests", "counter tests with increments other than one").

Every count is produced on the GPU by the fused generate-and-reduce kernels (nothing is
stored): one sq_fused_stats_ex run gives the top-16-bit histogram and the 32 per-bit ones
counts, a second run on the bit-reversed outputs gives (up to a fixed permutation) the
histogram of the low 16 bits, and sq_transitions counts adjacent differing bits.  From these
integers the host derives SPEC's desk battery: monobit, byte chi-square (df 255),
serial byte-pair chi-square (df 65535, non-overlapping little-endian pairs) and runs.

Stream convention: outputs u_0, u_1, ... of counters ctr0 + i*stride, little-endian 32-bit
words; bits LSB-first within a word; bytes b0..b3 of each word in address order.
Verdict: pass iff alpha <= p <= 1 - alpha (two-sided); runs reports
"dependent-failure" when the monobit proportion precondition fails.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_REV16 = None


def rev16_table() -> np.ndarray:
    """rev16[v] = the 16-bit reversal of v."""
    global _REV16
    if _REV16 is None:
        v = np.arange(65536, dtype=np.uint32)
        r = np.zeros(65536, dtype=np.uint32)
        for b in range(16):
            r |= ((v >> b) & 1) << (15 - b)
        _REV16 = r.astype(np.int64)
    return _REV16


@dataclass
class TestResult:
    name: str
    statistic: float
    p_value: float
    sample_bits: int
    verdict: str


def gpu_counts(key: int, ctr0: int, n: int, stride: int = 1, bitrev: bool = False, device=None) -> dict:
    """The integer counts of the stream, all computed by the CUDA kernels."""
    import torch

    from . import fused_stats_ex, transitions
    h_hi, ones = fused_stats_ex(key, ctr0, n, stride=stride, bitrev=bitrev, device=device)
    h_rev, _ = fused_stats_ex(key, ctr0, n, stride=stride, bitrev=not bitrev, device=device)
    tr = transitions(key, ctr0, n, stride=stride, bitrev=bitrev, device=device)
    torch.cuda.synchronize(h_hi.device)
    hist_hi = h_hi.cpu().numpy().view(np.uint64).astype(np.int64)
    hist_rev = h_rev.cpu().numpy().view(np.uint64).astype(np.int64)
    # hi16(bitrev(u)) = rev16(lo16(u)): hist_lo[v] = hist_rev[rev16(v)]
    hist_lo = hist_rev[rev16_table()]
    return {"n": n, "hist_hi": hist_hi, "hist_lo": hist_lo,
            "ones": ones.cpu().numpy().view(np.uint64).astype(np.int64),
            "transitions": int(tr.cpu().numpy().view(np.uint64)[0])}


def _chi2_p(chi2: float, df: int) -> float:
    from scipy.special import gammaincc
    return float(gammaincc(df / 2.0, chi2 / 2.0))


def _verdict(p: float, alpha: float) -> str:
    return "pass" if alpha <= p <= 1.0 - alpha else "fail"


def statistics(c: dict, alpha: float = 1e-6) -> list[TestResult]:
    n = int(c["n"])
    nbits = 32 * n
    S = int(np.asarray(c["ones"]).sum())
    res = []
    # monobit: |#ones - #zeros| / sqrt(n_bits), p = erfc(stat / sqrt(2))
    mono = abs(2 * S - nbits) / math.sqrt(nbits)
    p_mono = math.erfc(mono / math.sqrt(2.0))
    res.append(TestResult("monobit", mono, p_mono, nbits, _verdict(p_mono, alpha)))
    # byte chi-square: 4 bytes per word into 256 bins, df 255
    hh = np.asarray(c["hist_hi"]).reshape(256, 256)   # [b3][b2]
    hl = np.asarray(c["hist_lo"]).reshape(256, 256)   # [b1][b0]
    bytes_ = hh.sum(axis=0) + hh.sum(axis=1) + hl.sum(axis=0) + hl.sum(axis=1)
    e = 4.0 * n / 256.0
    chi_b = float(((bytes_ - e) ** 2).sum() / e)
    p_b = _chi2_p(chi_b, 255)
    res.append(TestResult("byte_chi_square", chi_b, p_b, nbits, _verdict(p_b, alpha)))
    # serial byte pairs: non-overlapping pairs (b0,b1), (b2,b3) -> 65536 bins, df 65535
    pairs = np.asarray(c["hist_hi"]) + np.asarray(c["hist_lo"])
    e = 2.0 * n / 65536.0
    chi_s = float(((pairs - e) ** 2).sum() / e)
    p_s = _chi2_p(chi_s, 65535)
    res.append(TestResult("serial_pair", chi_s, p_s, nbits, _verdict(p_s, alpha)))
    # runs: V = transitions + 1 vs 2 N pi (1 - pi) + 1
    pi = S / nbits
    if abs(pi - 0.5) >= 2.0 / math.sqrt(nbits):
        res.append(TestResult("runs", float("nan"), 0.0, nbits, "dependent-failure"))
    else:
        v = c["transitions"] + 1
        stat = abs(v - 2.0 * nbits * pi * (1.0 - pi)) / (2.0 * math.sqrt(2.0 * nbits) * pi * (1.0 - pi))
        p_r = math.erfc(stat)
        res.append(TestResult("runs", stat, p_r, nbits, _verdict(p_r, alpha)))
    return res


def run_battery(key: int, ctr0: int, n: int, stride: int = 1, bitrev: bool = False, alpha: float = 1e-6,
                device=None) -> list[TestResult]:
    """The desk battery on n squares32 outputs, computed on the GPU."""
    return statistics(gpu_counts(key, ctr0, n, stride, bitrev, device), alpha)


def scaled_uniformity(W: int, keys, device=None) -> list[tuple[float, float]]:
    """Exhaustive W-bit uniformity (the stand-in for P:17 footnote 1) on the
    GPU: for each key, every counter 0..2^W-1 of squares32_scaled, chi-square of the 2^(W/2)
    output counts against uniform; returns [(chi2, p), ...] (df = 2^(W/2) - 1)."""
    import torch

    from . import scaled_hist
    k = torch.tensor([int(x) & ((1 << 64) - 1) for x in keys], dtype=torch.uint64).view(torch.int64)
    k = k.to(device if device is not None else "cuda")
    out = []
    for s in range(0, k.numel(), 65535):
        h = scaled_hist(W, k[s:s + 65535].contiguous())
        torch.cuda.synchronize(h.device)
        h = h.cpu().numpy().view(np.uint64).astype(np.float64)
        e = float(1 << W) / h.shape[1]
        chi2 = ((h - e) ** 2).sum(axis=1) / e
        out += [(float(c), _chi2_p(float(c), h.shape[1] - 1)) for c in chi2]
    return out
