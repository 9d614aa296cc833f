"""Device plumbing: torch owns memory and streams, the C ABI does the work.

Every function here forwards raw device pointers and the current CUDA stream
to ``_smm_b200.so``; none of them computes anything on the host.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameterError


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("sketchmm_b200 needs a CUDA device (B200); there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise InvalidParameterError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def words_ptr(words: np.ndarray):
    words = np.ascontiguousarray(words, dtype=np.uint64)
    return words, words.ctypes.data_as(ctypes.c_void_p)


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def hash_table(hashes, group: int, n: int, device=None) -> torch.Tensor:
    """(d, n) uint32 buckets (group 0/1) or int8 signs (group 2/3) on the GPU."""
    lib = _lib.load()
    dev = require_cuda(device)
    d = hashes.d
    words, wp = words_ptr(hashes.packed_words())
    with torch.cuda.device(dev):
        if group < 2:
            out = torch.empty((d, n), dtype=torch.uint32, device=dev)
            _lib.check(lib.smm_hash_tables(wp, d, hashes.log2b, group, n, ptr(out), None, stream_ptr(dev)))
        else:
            out = torch.empty((d, n), dtype=torch.int8, device=dev)
            _lib.check(lib.smm_hash_tables(wp, d, hashes.log2b, group, n, None, ptr(out), stream_ptr(dev)))
    return out


def as_f64(x, device: torch.device) -> torch.Tensor:
    """Coerce numpy / torch input to a contiguous float64 CUDA tensor (copy only if needed)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float64)
    else:
        arr = np.asarray(x, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device=device, non_blocking=False)
    return t.contiguous()


def transpose(x: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    rows, cols = x.shape
    out = torch.empty((cols, rows), dtype=torch.float64, device=x.device)
    _lib.check(lib.smm_transpose(ptr(x), rows, cols, x.stride(0), ptr(out), rows, stream_ptr(x.device)))
    return out


def acc_shape(variant: str, d: int, b: int):
    return (d, b) if variant == "fwht" else (d, b // 2 + 1, 2)


KMAJOR = 0  # row k holds inner index k (the reference's A^T and B)
KMINOR = 1  # row i holds element i, inner index contiguous (A row-major, B^T row-major)


def _rowmajor(x: torch.Tensor) -> torch.Tensor:
    if x.dim() != 2 or x.dtype != torch.float64 or not x.is_cuda:
        raise InvalidParameterError("operands must be 2-D float64 CUDA tensors")
    if x.stride(1) != 1:
        x = x.contiguous()
    return x


def compress_accumulate(a: torch.Tensor, b: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str,
                        k0: int, k1: int, acc: torch.Tensor | None = None, a_layout: int = KMAJOR,
                        b_layout: int = KMAJOR) -> torch.Tensor:
    """Pre-inverse accumulator of inner indices [k0, k1).

    ``a`` is A^T (KMAJOR, rows = k) or A itself (KMINOR, columns = k); ``b`` is B
    (KMAJOR) or B^T (KMINOR).  Views with a row stride are used in place.
    """
    lib = _lib.load()
    a = _rowmajor(a)
    b = _rowmajor(b)
    dev = a.device
    n1 = a.shape[1] if a_layout == KMAJOR else a.shape[0]
    n2 = b.shape[1] if b_layout == KMAJOR else b.shape[0]
    v = _lib.VARIANT[variant]
    nbytes = ctypes.c_int64(0)
    _lib.check(lib.smm_compress_workspace_ex(v, d, log2b, n1, n2, k0, k1, a_layout, b_layout, ctypes.byref(nbytes)))
    ws = workspace(nbytes.value, dev)
    if acc is None:
        acc = torch.empty(acc_shape(variant, d, 1 << log2b), dtype=torch.float64, device=dev)
    words, wp = words_ptr(words)
    _lib.check(lib.smm_compress_accumulate_ex(v, ptr(a), a.stride(0), a_layout, ptr(b), b.stride(0), b_layout, n1,
                                              n2, k0, k1, wp, d, log2b, ptr(acc), ptr(ws), ws.numel(),
                                              stream_ptr(dev)))
    return acc


def finalize(acc: torch.Tensor, d: int, log2b: int, variant: str) -> torch.Tensor:
    lib = _lib.load()
    polys = torch.empty((d, 1 << log2b), dtype=torch.float64, device=acc.device)
    _lib.check(lib.smm_finalize(_lib.VARIANT[variant], ptr(acc), ptr(polys), d, log2b, stream_ptr(acc.device)))
    return polys


def extract(polys: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str, n1: int, n2: int,
            r0: int = 0, r1: int | None = None, want_est: bool = True, thr: float = 0.5, strict: bool = True,
            want_pairs: bool = False, est_out: torch.Tensor | None = None):
    """Rows [r0, r1) of the estimate grid and the heavy hitters |est| >(=) thr."""
    lib = _lib.load()
    dev = polys.device
    r1 = n1 if r1 is None else r1
    rows = r1 - r0
    nbytes = ctypes.c_int64(0)
    _lib.check(lib.smm_extract_workspace(d, n1, n2, r0, r1, ctypes.byref(nbytes)))
    ws = workspace(nbytes.value, dev)
    est = est_out
    if want_est and est is None:
        est = torch.empty((rows, n2), dtype=torch.float64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    words, wp = words_ptr(words)
    v = _lib.VARIANT[variant]
    ld = est.stride(0) if est is not None else n2
    _lib.check(lib.smm_extract(v, ptr(polys), wp, d, log2b, n1, n2, r0, r1, ptr(est), ld, float(thr),
                               1 if strict else 0, None, 0, ptr(count), ptr(ws), ws.numel(), stream_ptr(dev)))
    pairs = None
    if want_pairs:
        cnt = int(count.item())
        pairs = torch.empty((cnt, 2), dtype=torch.int64, device=dev)
        if cnt:
            # the bitmask of this extract call is still in `ws`: emit pairs without recomputing medians
            _lib.check(lib.smm_hh_pairs(ptr(ws), n2, r0, r1, ptr(pairs), cnt, stream_ptr(dev)))
    return est, count, pairs


def fwht_batched(x: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
    lib = _lib.load()
    n = x.shape[-1]
    log2n = n.bit_length() - 1
    batch = x.numel() // n if n else 0
    _lib.check(lib.smm_fwht_batched(ptr(x), batch, log2n, float(scale), stream_ptr(x.device)))
    return x


def fft_batched(z: torch.Tensor, inverse: bool = False, scale: float = 1.0) -> torch.Tensor:
    """z: complex128 CUDA tensor (..., n), transformed in place."""
    lib = _lib.load()
    n = z.shape[-1]
    log2n = n.bit_length() - 1
    batch = z.numel() // n if n else 0
    _lib.check(lib.smm_fft_batched(ptr(z), batch, log2n, 1 if inverse else 0, float(scale), stream_ptr(z.device)))
    return z
