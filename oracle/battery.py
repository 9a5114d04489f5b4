"""CPU oracle of the desk battery -- TEST INFRASTRUCTURE ONLY.

Works on the raw output stream (a numpy uint32 array of squares32 outputs from oracle.fill, or
any synthetic word stream for the pins): counts are taken directly from the stream's bits,
bytes and byte pairs (numpy unpackbits / bincount), p-values from the oracle's own regularized
incomplete gamma (oracle_gammaq) and math.erfc.  Shares nothing with the product's
paper_2004_06278_b200/battery.py, which derives the same counts from GPU histograms.
"""
from __future__ import annotations

import math

import numpy as np

import oracle as O


def counts(words: np.ndarray) -> dict:
    w = np.ascontiguousarray(words, dtype=np.uint32)
    b = w.view(np.uint8)                                   # little-endian bytes, address order
    bits = np.unpackbits(b, bitorder="little")            # LSB-first within each byte = within word
    return {
        "n": int(w.size),
        "ones_total": int(bits.sum()),
        "byte_hist": np.bincount(b, minlength=256).astype(np.int64),
        "pair_hist": np.bincount(w.view(np.uint16), minlength=65536).astype(np.int64),
        "transitions": int(np.count_nonzero(bits[1:] != bits[:-1])),
        "hist_hi": np.bincount(w >> np.uint32(16), minlength=65536).astype(np.int64),
    }


def _verdict(p, alpha):
    return "pass" if alpha <= p <= 1.0 - alpha else "fail"


def statistics(c: dict, alpha: float = 1e-6) -> dict:
    n = c["n"]
    nbits = 32 * n
    S = c["ones_total"]
    out = {}
    mono = abs(2 * S - nbits) / math.sqrt(nbits)
    p = math.erfc(mono / math.sqrt(2.0))
    out["monobit"] = (mono, p, _verdict(p, alpha))
    e = 4.0 * n / 256.0
    chi = float(((c["byte_hist"] - e) ** 2).sum() / e)
    p = O.gammaq(255 / 2.0, chi / 2.0)
    out["byte_chi_square"] = (chi, p, _verdict(p, alpha))
    e = 2.0 * n / 65536.0
    chi = float(((c["pair_hist"] - e) ** 2).sum() / e)
    p = O.gammaq(65535 / 2.0, chi / 2.0)
    out["serial_pair"] = (chi, p, _verdict(p, alpha))
    pi = S / nbits
    if abs(pi - 0.5) >= 2.0 / math.sqrt(nbits):
        out["runs"] = (float("nan"), 0.0, "dependent-failure")
    else:
        v = c["transitions"] + 1
        stat = abs(v - 2.0 * nbits * pi * (1.0 - pi)) / (2.0 * math.sqrt(2.0 * nbits) * pi * (1.0 - pi))
        p = math.erfc(stat)
        out["runs"] = (stat, p, _verdict(p, alpha))
    return out
