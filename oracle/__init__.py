"""ctypes binding of the plain CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product package
``paper_2004_06278_b200`` never imports it, and this module imports nothing from the product.

Every function forwards to the C transcription of the paper's listings (PAPER.md P:21-28,
P:56-64); see the header of oracle.c for what pins each one.  Arrays are numpy arrays; the
functions allocate their outputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

u64 = ctypes.c_uint64
u32 = ctypes.c_uint32
P = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no -march=native, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            sig = {
                "oracle_rot_half": (u64, [u64]),
                "oracle_round": (u64, [u64, u64]),
                "oracle_squares32": (u32, [u64, u64]),
                "oracle_squares64": (u64, [u64, u64]),
                "oracle_squares32_limb": (u32, [u64, u64]),
                "oracle_squares64_limb": (u64, [u64, u64]),
                "oracle_squares32_i128": (u32, [u64, u64]),
                "oracle_squares64_i128": (u64, [u64, u64]),
                "oracle_squares32_pairs": (None, [P, P, u64, P]),
                "oracle_squares64_pairs": (None, [P, P, u64, P]),
                "oracle_squares32_pairs_limb": (None, [P, P, u64, P]),
                "oracle_squares64_pairs_limb": (None, [P, P, u64, P]),
                "oracle_squares32_pairs_i128": (None, [P, P, u64, P]),
                "oracle_squares64_pairs_i128": (None, [P, P, u64, P]),
                "oracle_fill_u32": (None, [P, u64, u64, u64, P, u64]),
                "oracle_fill_u64": (None, [P, u64, u64, u64, P, u64]),
                "oracle_fill_f32": (None, [P, u64, u64, u64, P, u64]),
                "oracle_f32_from_u32": (ctypes.c_float, [u32]),
                "oracle_fused_stats": (None, [u64, u64, u64, P, P]),
                "oracle_f64_from_u64": (ctypes.c_double, [u64]),
                "oracle_fill_f64": (None, [P, u64, u64, u64, P, u64]),
                "oracle_fill_f32x2": (None, [P, u64, u64, u64, P, u64]),
                "oracle_fill_strided": (None, [ctypes.c_int, P, u64, u64, u64, u64, P, u64]),
                "oracle_fill_keyctr": (None, [ctypes.c_int, P, u64, u64, P]),
                "oracle_bitrev32": (u32, [u32]),
                "oracle_fused_stats_ex": (None, [u64, u64, u64, u64, ctypes.c_int, P, P]),
                "oracle_xorfold_u32": (u64, [u64, u64, u64]),
                "oracle_weyl_check": (ctypes.c_int, [u64, u64]),
                "oracle_validate_key": (u32, [u64]),
                "oracle_key_candidate": (u64, [u64, u64, u64]),
                "oracle_keygen": (ctypes.c_int, [u64, u64, P]),
                "oracle_squares32_scaled": (u64, [u64, u64, ctypes.c_int]),
                "oracle_gammaq": (ctypes.c_double, [ctypes.c_double, ctypes.c_double]),
                "oracle_scaled_hist_range": (None, [u64, ctypes.c_int, u64, u64, P]),
                "oracle_scaled_uniformity": (ctypes.c_int, [u64, ctypes.c_int,
                                                             ctypes.POINTER(ctypes.c_double),
                                                             ctypes.POINTER(ctypes.c_double)]),
                "oracle_partition": (ctypes.c_int, [u64, u64, u64, u64] + [ctypes.POINTER(u64)] * 4),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


M64 = (1 << 64) - 1

# Key-rule bits of oracle_validate_key.
KEY_UPPER_REPEAT, KEY_LOWER_REPEAT, KEY_ZERO_DIGIT, KEY_EVEN, KEY_POPCOUNT = 1, 2, 4, 8, 16


# ---------------------------------------------------------------- scalar transcriptions
def rot_half(x: int) -> int:
    return lib().oracle_rot_half(x & M64)


def round_(x: int, w: int) -> int:
    return lib().oracle_round(x & M64, w & M64)


def squares32(ctr: int, key: int) -> int:
    return lib().oracle_squares32(ctr & M64, key & M64)


def squares64(ctr: int, key: int) -> int:
    return lib().oracle_squares64(ctr & M64, key & M64)


def squares32_limb(ctr: int, key: int) -> int:
    return lib().oracle_squares32_limb(ctr & M64, key & M64)


def squares64_limb(ctr: int, key: int) -> int:
    return lib().oracle_squares64_limb(ctr & M64, key & M64)


def squares32_i128(ctr: int, key: int) -> int:
    return lib().oracle_squares32_i128(ctr & M64, key & M64)


def squares64_i128(ctr: int, key: int) -> int:
    return lib().oracle_squares64_i128(ctr & M64, key & M64)


def squares_pairs(ctr: np.ndarray, key: np.ndarray, width: int = 32, method: str = "listing") -> np.ndarray:
    """Evaluate over explicit (ctr[i], key[i]) pairs.  method: listing | limb | i128."""
    ctr = np.ascontiguousarray(ctr, dtype=np.uint64)
    key = np.ascontiguousarray(key, dtype=np.uint64)
    assert ctr.shape == key.shape
    out = np.empty(ctr.shape, dtype=np.uint32 if width == 32 else np.uint64)
    suffix = {"listing": "", "limb": "_limb", "i128": "_i128"}[method]
    fn = getattr(lib(), f"oracle_squares{width}_pairs{suffix}")
    fn(_ptr(ctr), _ptr(key), ctr.size, _ptr(out))
    return out


# ---------------------------------------------------------------- fills and statistics
def _keys_array(keys) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))


KIND_CODE = {"u32": 0, "u64": 1, "f32": 2, "f64": 3, "f32x2": 4}
KIND_DTYPE = {"u32": np.uint32, "u64": np.uint64, "f32": np.float32, "f64": np.float64, "f32x2": np.float32}


def fill(kind: str, keys, ctr0: int, n: int, ld: int | None = None) -> np.ndarray:
    """out[k, i] = G(ctr0 + i mod 2^64, keys[k]) for kind in u32 | u64 | f32 | f64 | f32x2;
    shape (nkeys, ld) (f32x2: (nkeys, ld, 2), low half first)."""
    ka = _keys_array(keys)
    ld = n if ld is None else ld
    shape = (ka.size, ld, 2) if kind == "f32x2" else (ka.size, ld)
    out = np.zeros(shape, dtype=KIND_DTYPE[kind])
    getattr(lib(), f"oracle_fill_{kind}")(_ptr(ka), ka.size, ctr0 & M64, n, _ptr(out), ld)
    return out


def fill_strided(kind: str, keys, ctr0: int, stride: int, n: int, ld: int | None = None) -> np.ndarray:
    """Raw element bits (uint32 for u32/f32, uint64 otherwise) of the strided fill."""
    ka = _keys_array(keys)
    ld = n if ld is None else ld
    out = np.zeros((ka.size, ld), dtype=np.uint32 if kind in ("u32", "f32") else np.uint64)
    lib().oracle_fill_strided(KIND_CODE[kind], _ptr(ka), ka.size, ctr0 & M64, stride & M64, n, _ptr(out), ld)
    return out


def fill_keyctr(kind: str, keys, ctr: int) -> np.ndarray:
    """Raw element bits of G(ctr, keys[j]) for every key j (key-counter mode)."""
    ka = _keys_array(keys)
    out = np.zeros(ka.size, dtype=np.uint32 if kind in ("u32", "f32") else np.uint64)
    lib().oracle_fill_keyctr(KIND_CODE[kind], _ptr(ka), ka.size, ctr & M64, _ptr(out))
    return out


def f64_from_u64(v: int) -> float:
    return lib().oracle_f64_from_u64(v & M64)


def bitrev32(u: int) -> int:
    return lib().oracle_bitrev32(u & 0xFFFFFFFF)


def fused_stats_ex(key: int, ctr0: int, stride: int, n: int, bitrev: bool = False):
    hist = np.zeros(65536, dtype=np.uint64)
    ones = np.zeros(32, dtype=np.uint64)
    lib().oracle_fused_stats_ex(key & M64, ctr0 & M64, stride & M64, n, int(bitrev), _ptr(hist), _ptr(ones))
    return hist, ones


def f32_from_u32(u: int) -> float:
    return lib().oracle_f32_from_u32(u)


def fused_stats(key: int, ctr0: int, n: int, hist: np.ndarray | None = None,
                ones: np.ndarray | None = None):
    """Accumulate hist[65536] and ones[32] (uint64) over squares32(ctr0 .. ctr0+n-1, key)."""
    hist = np.zeros(65536, dtype=np.uint64) if hist is None else hist
    ones = np.zeros(32, dtype=np.uint64) if ones is None else ones
    assert hist.dtype == np.uint64 and hist.size == 65536 and hist.flags.c_contiguous
    assert ones.dtype == np.uint64 and ones.size == 32 and ones.flags.c_contiguous
    lib().oracle_fused_stats(key & M64, ctr0 & M64, n, _ptr(hist), _ptr(ones))
    return hist, ones


def xorfold_u32(key: int, ctr0: int, n: int) -> int:
    return lib().oracle_xorfold_u32(key & M64, ctr0 & M64, n)


def weyl_check(s: int, n: int) -> bool:
    return bool(lib().oracle_weyl_check(s & M64, n))


# ---------------------------------------------------------------- keys
def validate_key(key: int) -> int:
    return lib().oracle_validate_key(key & M64)


def key_candidate(seed: int, j: int, attempt: int) -> int:
    return lib().oracle_key_candidate(seed & M64, j, attempt)


def keygen(seed: int, count: int) -> np.ndarray:
    out = np.zeros(max(count, 1), dtype=np.uint64)
    rc = lib().oracle_keygen(seed & M64, count, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_keygen failed with code {rc}")
    return out[:count]


# ---------------------------------------------------------------- scaled analogue, partition
def squares32_scaled(ctr: int, key: int, W: int) -> int:
    return lib().oracle_squares32_scaled(ctr & M64, key & M64, W)


def scaled_hist_range(key: int, W: int, c0: int, n: int, hist: np.ndarray | None = None) -> np.ndarray:
    hist = np.zeros(1 << (W // 2), dtype=np.uint64) if hist is None else hist
    lib().oracle_scaled_hist_range(key & M64, W, c0, n, _ptr(hist))
    return hist


def gammaq(a: float, x: float) -> float:
    return lib().oracle_gammaq(a, x)


def scaled_uniformity(key: int, W: int):
    chi2, p = ctypes.c_double(), ctypes.c_double()
    rc = lib().oracle_scaled_uniformity(key & M64, W, ctypes.byref(chi2), ctypes.byref(p))
    if rc != 0:
        raise ValueError("bad W")
    return chi2.value, p.value


def partition(n: int, parts: int, idx: int):
    """(start, length) of part idx of [0, n) split into `parts`; n may be 2**64."""
    sh, sl, lh, ll = u64(), u64(), u64(), u64()
    rc = lib().oracle_partition(n >> 64, n & M64, parts, idx, ctypes.byref(sh), ctypes.byref(sl),
                                ctypes.byref(lh), ctypes.byref(ll))
    if rc != 0:
        raise ValueError("bad partition arguments")
    return (sh.value << 64) | sl.value, (lh.value << 64) | ll.value
