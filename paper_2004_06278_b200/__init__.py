"""paper_2004_06278_b200 -- B200 (sm_100a) bulk evaluator of the Squares counter-based RNG
(B. Widynski, arXiv 2004.06278).

Thin Python binding of ``libsquares.so`` (C ABI in ``include/squares.h``): argument
marshalling only.  Every step of the hot path runs in the library's CUDA kernels; there is no
CPU or PyTorch fallback -- if the extension is missing or a call fails, these functions raise.

PyTorch supplies device memory (tensors), the current CUDA stream and process groups.
Tensor dtypes: keys are int64 tensors (reinterpreted as uint64); u32 outputs are int32
(reinterpreted as uint32), u64 outputs int64, f32 outputs float32.  Fused counts are int64
tensors (uint64 counts; NCCL SUM over int64 is bit-identical to uint64 addition mod 2^64).
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import dist  # noqa: F401  (multi-GPU composition: partition + NCCL all-reduce)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsquares.so")
# SQ_LIB: load an experimental build of the same library instead (tools/build_variant.sh);
# unset for the product path.
LIB_PATH = os.environ.get("SQ_LIB", LIB_PATH)

SQ_OK, SQ_EINVAL, SQ_ERANGE, SQ_ECUDA, SQ_ENOMEM = 0, 1, 2, 3, 4
KEY_UPPER_REPEAT, KEY_LOWER_REPEAT, KEY_ZERO_DIGIT, KEY_EVEN, KEY_POPCOUNT = 1, 2, 4, 8, 16
KINDS = {"u32": 0, "u64": 1, "f32": 2, "f64": 3, "f32x2": 4}
SQ_FUSED_BITREV = 1
HIST_BINS = 65536
M64 = (1 << 64) - 1

_lib = None


class SquaresError(RuntimeError):
    def __init__(self, fn: str, code: int):
        lib = _load()
        msg = lib.sq_strerror(code).decode()
        if code == SQ_ECUDA:
            msg += f" (cudaError {lib.sq_last_cuda_error()})"
        super().__init__(f"{fn}: {msg}")
        self.code = code


def _load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2004_06278_b200._build` "
            "(or __graft_entry__.build()); there is no fallback implementation")
    L = ctypes.CDLL(LIB_PATH)
    u64, u32, vp, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
    sigs = {
        "sq_strerror": (ctypes.c_char_p, [i32]),
        "sq_last_cuda_error": (i32, []),
        "sq_version": (i32, []),
        "sq_validate_key": (u32, [u64]),
        "sq_keygen": (i32, [u64, u64, vp]),
        "sq_fill_u32": (i32, [vp, u64, u64, u64, vp, u64, vp]),
        "sq_fill_u64": (i32, [vp, u64, u64, u64, vp, u64, vp]),
        "sq_fill_f32": (i32, [vp, u64, u64, u64, vp, u64, vp]),
        "sq_fill_u32_k": (i32, [u64, u64, u64, vp, vp]),
        "sq_fill_u64_k": (i32, [u64, u64, u64, vp, vp]),
        "sq_fill_f32_k": (i32, [u64, u64, u64, vp, vp]),
        "sq_fill_f64": (i32, [vp, u64, u64, u64, vp, u64, vp]),
        "sq_fill_f32x2": (i32, [vp, u64, u64, u64, vp, u64, vp]),
        "sq_fill_f64_k": (i32, [u64, u64, u64, vp, vp]),
        "sq_fill_f32x2_k": (i32, [u64, u64, u64, vp, vp]),
        "sq_fill_ex": (i32, [i32, vp, u64, u64, u64, u64, u64, vp, u64, vp]),
        "sq_fill_keyctr": (i32, [i32, vp, u64, u64, vp, vp]),
        "sq_fused_stats": (i32, [u64, u64, u64, vp, vp, vp]),
        "sq_fused_stats_ex": (i32, [u64, u64, u64, u64, u32, vp, vp, vp]),
        "sq_transitions": (i32, [u64, u64, u64, u64, u32, vp, vp]),
        "sq_scaled_hist": (i32, [i32, vp, u64, vp, vp]),
        "sq_fill_host": (i32, [i32, u64, u64, u64, vp, vp, ctypes.c_size_t, vp, vp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED_SYMBOLS = ("sq_strerror", "sq_last_cuda_error", "sq_version", "sq_validate_key", "sq_keygen",
                    "sq_fill_u32", "sq_fill_u64", "sq_fill_f32", "sq_fill_u32_k", "sq_fill_u64_k",
                    "sq_fill_f32_k", "sq_fill_f64", "sq_fill_f32x2", "sq_fill_f64_k", "sq_fill_f32x2_k", "sq_fill_ex", "sq_fill_keyctr",
                    "sq_fused_stats", "sq_fused_stats_ex", "sq_transitions", "sq_scaled_hist", "sq_fill_host")


def _check(fn: str, code: int) -> None:
    if code != SQ_OK:
        raise SquaresError(fn, code)


def _device(dev) -> torch.device:
    """A concrete CUDA device (index resolved) from a tensor device, a string or None."""
    d = torch.device(dev if dev is not None else "cuda")
    if d.type != "cuda":
        raise ValueError(f"expected a CUDA device, got {d}")
    return torch.device("cuda", torch.cuda.current_device() if d.index is None else d.index)


def _stream_handle(stream, device: torch.device | None = None) -> int:
    """The raw stream the library launches on: `stream`, else `device`'s current stream.  The
    C ABI launches on the CURRENT device, so every entry point below runs inside
    `torch.cuda.device(device)` and a stream of another device is rejected."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    elif device is not None and stream.device != device:
        raise ValueError(f"stream is on {stream.device}, tensors on {device}")
    return stream.cuda_stream


def _u64(x: int) -> int:
    return int(x) & M64


def _count(n: int, what: str = "n") -> int:
    """A count argument of the C ABI (uint64): 0 <= n < 2^64, else ValueError (ctypes would
    silently reduce it mod 2^64)."""
    n = int(n)
    if not 0 <= n <= M64:
        raise ValueError(f"{what} = {n} is outside [0, 2^64)")
    return n


def _check_keys(keys: torch.Tensor) -> torch.device:
    if not (isinstance(keys, torch.Tensor) and keys.is_cuda and keys.dtype == torch.int64 and keys.dim() == 1
            and keys.is_contiguous()):
        raise ValueError("keys must be a contiguous 1-D int64 CUDA tensor")
    return _device(keys.device)


def _check_counts(t: torch.Tensor, numel: int, name: str, device: torch.device | None) -> torch.device:
    """Caller-supplied accumulators (hist / ones / count): the kernels atomically add to exactly
    `numel` uint64 entries, so anything else would be an out-of-bounds device write."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64 and t.numel() == numel
            and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous int64 CUDA tensor of {numel} elements")
    d = _device(t.device)
    if device is not None and d != device:
        raise ValueError(f"{name} is on {d}, expected {device}")
    return d


# ----------------------------------------------------------------------------- host functions
def version() -> int:
    return _load().sq_version()


def validate_key(key: int) -> int:
    """Bitmask of violated key rules (0 = valid); see include/squares.h."""
    return _load().sq_validate_key(_u64(key))


def keygen(seed: int, count: int) -> torch.Tensor:
    """`count` keys of stream `seed` (documented "different digits" mapping), int64 CPU tensor."""
    count = _count(count, "count")
    if count > (1 << 31):   # the library's SQ_ERANGE, checked before allocating count keys
        raise SquaresError("sq_keygen", SQ_ERANGE)
    out = torch.empty(max(count, 1), dtype=torch.int64)
    _check("sq_keygen", _load().sq_keygen(_u64(seed), count, out.data_ptr()))
    return out[: int(count)]


# ----------------------------------------------------------------------------- device functions
# element dtypes; an f32x2 element is a PAIR of float32 (low half of squares64 first), so its
# tensors have a trailing dimension of 2.
_OUT_DTYPE = {"u32": torch.int32, "u64": torch.int64, "f32": torch.float32, "f64": torch.float64,
              "f32x2": torch.float32}
_ELEM_BYTES = {"u32": 4, "u64": 8, "f32": 4, "f64": 8, "f32x2": 8}


def _alloc(kind, shape, device):
    if kind == "f32x2":
        shape = tuple(shape) + (2,)
    return torch.empty(shape, dtype=_OUT_DTYPE[kind], device=device)


def _elems(kind, t: torch.Tensor) -> int:
    return t.numel() * t.element_size() // _ELEM_BYTES[kind]


def _check_out(kind: str, out: torch.Tensor, need: int, device: torch.device) -> None:
    if not (isinstance(out, torch.Tensor) and out.dtype == _OUT_DTYPE[kind] and out.is_cuda
            and out.is_contiguous()):
        raise ValueError(f"out must be a contiguous CUDA {_OUT_DTYPE[kind]} tensor")
    if _device(out.device) != device:
        raise ValueError(f"out is on {out.device}, expected {device}")
    if _elems(kind, out) < need:
        raise ValueError(f"out holds {_elems(kind, out)} elements, {need} needed")


def _infer_ld(kind: str, out: torch.Tensor | None, ld: int | None, n: int) -> int:
    """Row pitch: explicit `ld`, else the row length of a 2-D out (3-D for f32x2), else n."""
    if ld is not None:
        return _count(ld, "ld")
    nd = 3 if kind == "f32x2" else 2
    if out is not None and out.dim() == nd:
        return int(out.shape[1])
    return n


def _fill(kind: str, keys: torch.Tensor, ctr0: int, n: int, out: torch.Tensor | None, ld: int | None,
          stream=None) -> torch.Tensor:
    dev = _check_keys(keys)
    n = _count(n)
    nkeys = keys.numel()
    ld = _infer_ld(kind, out, ld, n)
    if out is None:
        out = _alloc(kind, (nkeys, ld), dev)
    else:
        _check_out(kind, out, (nkeys - 1) * ld + n if nkeys else 0, dev)
    fn = getattr(_load(), f"sq_fill_{kind}")
    with torch.cuda.device(dev):
        _check(f"sq_fill_{kind}", fn(keys.data_ptr(), nkeys, _u64(ctr0), n, out.data_ptr(), ld,
                                     _stream_handle(stream, dev)))
    return out


def _fill_k(kind: str, key: int, ctr0: int, n: int, out: torch.Tensor | None, device=None,
            stream=None) -> torch.Tensor:
    n = _count(n)
    if out is None:
        dev = _device(device)
        out = _alloc(kind, (n,), dev)
    else:
        dev = _device(out.device)
        if device is not None and _device(device) != dev:
            raise ValueError(f"out is on {dev}, device={device}")
        _check_out(kind, out, n, dev)
    fn = getattr(_load(), f"sq_fill_{kind}_k")
    with torch.cuda.device(dev):
        _check(f"sq_fill_{kind}_k", fn(_u64(key), _u64(ctr0), n, out.data_ptr(), _stream_handle(stream, dev)))
    return out


def fill_u32_k(key, ctr0, n, out=None, device=None, stream=None):
    """Single-key fill, key by value: out[i] = squares32(ctr0 + i, key)."""
    return _fill_k("u32", key, ctr0, n, out, device, stream)


def fill_u64_k(key, ctr0, n, out=None, device=None, stream=None):
    """Single-key fill, key by value: out[i] = squares64(ctr0 + i, key)."""
    return _fill_k("u64", key, ctr0, n, out, device, stream)


def fill_f32_k(key, ctr0, n, out=None, device=None, stream=None):
    """Single-key fill, key by value: out[i] = (squares32(ctr0 + i, key) >> 8) * 2^-24."""
    return _fill_k("f32", key, ctr0, n, out, device, stream)


def fill_u32(keys, ctr0, n, out=None, ld=None, stream=None):
    """out[k, i] = squares32(ctr0 + i, keys[k]) as int32 bit patterns."""
    return _fill("u32", keys, ctr0, n, out, ld, stream)


def fill_u64(keys, ctr0, n, out=None, ld=None, stream=None):
    """out[k, i] = squares64(ctr0 + i, keys[k]) as int64 bit patterns."""
    return _fill("u64", keys, ctr0, n, out, ld, stream)


def fill_f32(keys, ctr0, n, out=None, ld=None, stream=None):
    """out[k, i] = (squares32(ctr0 + i, keys[k]) >> 8) * 2^-24, float32 in [0, 1)."""
    return _fill("f32", keys, ctr0, n, out, ld, stream)


def fill_f64(keys, ctr0, n, out=None, ld=None, stream=None):
    """out[k, i] = (squares64(ctr0 + i, keys[k]) >> 11) * 2^-53, float64 in [0, 1)."""
    return _fill("f64", keys, ctr0, n, out, ld, stream)


def fill_f32x2(keys, ctr0, n, out=None, ld=None, stream=None):
    """out[k, i, :] = the two 32-bit halves of squares64(ctr0 + i, keys[k]) as floats
    (h >> 8) * 2^-24, low half first."""
    return _fill("f32x2", keys, ctr0, n, out, ld, stream)


def fill_f64_k(key, ctr0, n, out=None, device=None, stream=None):
    return _fill_k("f64", key, ctr0, n, out, device, stream)


def fill_f32x2_k(key, ctr0, n, out=None, device=None, stream=None):
    return _fill_k("f32x2", key, ctr0, n, out, device, stream)


def fill_ex(kind: str, ctr0: int, n: int, stride: int = 1, keys: torch.Tensor | None = None,
            key: int | None = None, out: torch.Tensor | None = None, ld: int | None = None,
            device=None, stream=None) -> torch.Tensor:
    """Generic fill (sq_fill_ex): counters ctr0 + i*stride; either a device keys tensor
    (rows) or one key by value."""
    if (keys is None) == (key is None):
        raise ValueError("pass exactly one of keys (device tensor) or key (int)")
    n = _count(n)
    if keys is not None:
        dev = _check_keys(keys)
        nkeys, kptr, kimm = keys.numel(), keys.data_ptr(), 0
    else:
        dev = _device(out.device if out is not None and device is None else device)
        nkeys, kptr, kimm = 1, None, _u64(key)
    ld = _infer_ld(kind, out, ld, n)
    if out is None:
        out = _alloc(kind, (nkeys, ld), dev)
    else:
        _check_out(kind, out, (nkeys - 1) * ld + n if nkeys else 0, dev)
    with torch.cuda.device(dev):
        _check("sq_fill_ex", _load().sq_fill_ex(KINDS[kind], kptr, nkeys, kimm, _u64(ctr0), _u64(stride), n,
                                                out.data_ptr(), ld, _stream_handle(stream, dev)))
    return out


def fill_keyctr(kind: str, keys: torch.Tensor, ctr: int, out: torch.Tensor | None = None, stream=None):
    """Key-counter mode: out[j] = G(ctr, keys[j])."""
    dev = _check_keys(keys)
    if out is None:
        out = _alloc(kind, (keys.numel(),), dev)
    else:
        _check_out(kind, out, keys.numel(), dev)
    with torch.cuda.device(dev):
        _check("sq_fill_keyctr", _load().sq_fill_keyctr(KINDS[kind], keys.data_ptr(), keys.numel(), _u64(ctr),
                                                        out.data_ptr(), _stream_handle(stream, dev)))
    return out


def _zeros(shape, dev, stream):
    """Zeroed int64 counts, the memset enqueued on `stream` (the stream the kernel will run on)
    so that it is ordered before the accumulating kernel even when `stream` is not current."""
    if stream is None:
        return torch.zeros(shape, dtype=torch.int64, device=dev)
    _stream_handle(stream, dev)   # a stream of another device is rejected here already
    with torch.cuda.stream(stream):
        return torch.zeros(shape, dtype=torch.int64, device=dev)


def _counts_pair(hist, ones, device, stream=None):
    """(hist, ones, device): allocated zeroed on `device` when None, else validated."""
    dev = None
    if hist is not None:
        dev = _check_counts(hist, HIST_BINS, "hist", None)
    if ones is not None:
        dev = _check_counts(ones, 32, "ones", dev)
    if dev is None:
        dev = _device(device)
    elif device is not None and _device(device) != dev:
        raise ValueError(f"counts are on {dev}, device={device}")
    if hist is None:
        hist = _zeros(HIST_BINS, dev, stream)
    if ones is None:
        ones = _zeros(32, dev, stream)
    return hist, ones, dev


def fused_stats_ex(key: int, ctr0: int, n: int, stride: int = 1, bitrev: bool = False,
                   hist: torch.Tensor | None = None, ones: torch.Tensor | None = None, device=None, stream=None):
    """Fused statistics over counters ctr0 + i*stride, optionally of bit-reversed outputs."""
    n = _count(n)
    hist, ones, dev = _counts_pair(hist, ones, device, stream)
    with torch.cuda.device(dev):
        _check("sq_fused_stats_ex", _load().sq_fused_stats_ex(_u64(key), _u64(ctr0), _u64(stride), n,
                                                              SQ_FUSED_BITREV if bitrev else 0, hist.data_ptr(),
                                                              ones.data_ptr(), _stream_handle(stream, dev)))
    return hist, ones


def transitions(key: int, ctr0: int, n: int, stride: int = 1, bitrev: bool = False,
                count: torch.Tensor | None = None, device=None, stream=None) -> torch.Tensor:
    """Accumulate the number of adjacent differing bits of the LSB-first output bit stream."""
    n = _count(n)
    if count is None:
        dev = _device(device)
        count = _zeros(1, dev, stream)
    else:
        dev = _check_counts(count, 1, "count", _device(device) if device is not None else None)
    with torch.cuda.device(dev):
        _check("sq_transitions", _load().sq_transitions(_u64(key), _u64(ctr0), _u64(stride), n,
                                                        SQ_FUSED_BITREV if bitrev else 0, count.data_ptr(),
                                                        _stream_handle(stream, dev)))
    return count


def scaled_hist(W: int, keys: torch.Tensor, hist: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exhaustive W-bit uniformity histograms, shape (nkeys, 2^(W/2)) int64 (accumulating)."""
    dev = _check_keys(keys)
    if not (isinstance(W, int) and 8 <= W <= 32 and W % 2 == 0):
        raise ValueError("W must be an even integer in [8, 32]")
    nb = 1 << (W // 2)
    if hist is None:
        hist = _zeros((keys.numel(), nb), dev, stream)
    else:
        _check_counts(hist, keys.numel() * nb, "hist", dev)
    with torch.cuda.device(dev):
        _check("sq_scaled_hist", _load().sq_scaled_hist(int(W), keys.data_ptr(), keys.numel(), hist.data_ptr(),
                                                        _stream_handle(stream, dev)))
    return hist


def fused_stats(key: int, ctr0: int, n: int, hist: torch.Tensor | None = None,
                ones: torch.Tensor | None = None, device=None, stream=None):
    """Accumulate the top-16-bit histogram (65536 bins) and the 32 per-bit ones counts of
    squares32 over [ctr0, ctr0 + n) into int64 CUDA tensors (allocated zeroed if None)."""
    n = _count(n)
    hist, ones, dev = _counts_pair(hist, ones, device, stream)
    with torch.cuda.device(dev):
        _check("sq_fused_stats", _load().sq_fused_stats(_u64(key), _u64(ctr0), n, hist.data_ptr(),
                                                        ones.data_ptr(), _stream_handle(stream, dev)))
    return hist, ones


def fill_host(kind: str, key: int, ctr0: int, n: int, out_host: torch.Tensor, scratch: torch.Tensor,
              stream=None, copy_stream=None) -> torch.Tensor:
    """End-to-end fill of ONE key into a (pinned) host tensor via the library's chunked
    generate + D2H pipeline.  Synchronous."""
    n = _count(n)
    es = _ELEM_BYTES[kind]
    if out_host.is_cuda or out_host.numel() * out_host.element_size() < n * es:
        raise ValueError("out_host must be a host tensor of at least n elements")
    if not (scratch.is_cuda and scratch.is_contiguous()):
        raise ValueError("scratch must be a contiguous CUDA tensor")
    dev = _device(scratch.device)
    with torch.cuda.device(dev):
        cs = _stream_handle(copy_stream, dev) if copy_stream is not None else None
        _check("sq_fill_host", _load().sq_fill_host(KINDS[kind], _u64(key), _u64(ctr0), n,
                                                    out_host.data_ptr(), scratch.data_ptr(),
                                                    scratch.numel() * scratch.element_size(),
                                                    _stream_handle(stream, dev), cs))
    return out_host


def as_unsigned(t: torch.Tensor):
    """numpy view of an int32/int64 CPU tensor as uint32/uint64."""
    import numpy as np
    a = t.numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a.view(np.uint64) if a.dtype == np.int64 else a
