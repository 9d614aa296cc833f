"""Public sketched-product API — a drop-in for the reference ``sketchmm.sketch``.

Same names, argument meaning, validation and exceptions as the reference
(sketch.py:58-494, exported at __init__.py:9-75).  The difference is where the
work runs: hashing tables, compression (steps 1-3), the inverse transform
(step 4) and extraction + heavy-hitter threshold (step 5) all execute in the
sm_100a kernels of ``_smm_b200.so``; inputs may be host arrays (numpy or CPU
tensors: streamed to the GPU in k-slabs that overlap the kernel) or CUDA
tensors (used in place when float64).  There is no CPU fallback: without the
extension or a GPU every hot-path call raises.

Reference behaviour kept on purpose:
  * validation happens before any kernel work (sketch.py:68-82, 266-301, 335-355);
  * hash functions are drawn from ``default_rng(params.seed)`` in the reference
    order, so bucket/sign assignments are bit-identical;
  * ``threads`` is validated like ``effective_threads`` (sketch.py:108-114) but
    does not change the result: the GPU reduction order is fixed by the kernel
    geometry, so runs are bit-identical regardless of ``threads``.
"""

from __future__ import annotations

import functools
import math
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import FormatError, InvalidParameterError
from .hashing import HashPair, SketchHashes, check_buckets, eval_bucket, eval_sign

TRANSFORMS = ("fft", "fwht")
TRANSFORM_CODES = {"fft": 0, "fwht": 1}
TRANSFORM_NAMES = {v: k for k, v in TRANSFORM_CODES.items()}
SKETCH_MAGIC = b"SKCH"
SKETCH_VERSION = 1
SKETCH_HEADER = struct.Struct("<4sIQQQIQ")
MAX_BUCKETS = 1 << 32
MAX_SEED = (1 << 64) - 1


def _is_pow2(v: int) -> bool:
    return v >= 1 and (v & (v - 1)) == 0


@dataclass(frozen=True)
class SketchParams:
    """Sketch configuration (sketch.py:58-82)."""

    n: int
    b: int
    d: int
    transform: str = "fwht"
    seed: int = 0

    def __post_init__(self) -> None:
        if not (isinstance(self.n, (int, np.integer)) and self.n >= 1):
            raise InvalidParameterError(f"n must be a positive integer, got {self.n}")
        if not (isinstance(self.b, (int, np.integer)) and 2 <= self.b <= MAX_BUCKETS and _is_pow2(int(self.b))):
            raise InvalidParameterError(f"b must be a power of two in [2, 2**32], got {self.b}")
        if not (isinstance(self.d, (int, np.integer)) and self.d >= 1 and self.d % 2 == 1):
            raise InvalidParameterError(f"d must be an odd positive integer, got {self.d}")
        if self.transform not in TRANSFORMS:
            raise InvalidParameterError(f"transform must be one of {TRANSFORMS}, got {self.transform!r}")
        if not (0 <= int(self.seed) <= MAX_SEED):
            raise InvalidParameterError("seed must fit in 64 bits")

    @property
    def log2b(self) -> int:
        return int(self.b).bit_length() - 1


def derive_params(n: int, c_d: float, c_b: float, transform: str = "fwht", seed: int = 0) -> SketchParams:
    """d = 2*floor(c_d*log2(n)/2) + 1, b = c_b*n (sketch.py:85-105)."""
    if not (isinstance(n, (int, np.integer)) and n >= 2 and _is_pow2(int(n))):
        raise InvalidParameterError(f"n must be a power of two >= 2, got {n}")
    if not (c_d > 0 and c_b > 0):
        raise InvalidParameterError("c_d and c_b must be positive")
    logn = int(n).bit_length() - 1
    d = 2 * math.floor(c_d * logn / 2.0) + 1
    b_float = c_b * n
    b = int(round(b_float))
    if abs(b_float - b) > 1e-9 * max(b, 1) or not _is_pow2(b) or b < 2:
        raise InvalidParameterError(f"c_b * n must be a power of two >= 2, got {b_float!r}")
    return SketchParams(n=int(n), b=b, d=d, transform=transform, seed=int(seed))


def effective_threads(threads: int | None = None) -> int:
    """Validated like the reference (sketch.py:108-114); no effect on results."""
    if threads is None:
        return 1
    if not (isinstance(threads, (int, np.integer)) and threads >= 1):
        raise InvalidParameterError(f"threads must be a positive integer, got {threads}")
    return int(threads)


class ProductSketch:
    """Compressed representation of one matrix product (sketch.py:123-149).

    ``polys`` is the (d, b) float64 sketch as a numpy array (a host copy of the
    device tensor, made on first access); ``polys_device()`` returns the CUDA
    tensor.  Assigning or mutating the numpy ``polys`` makes it authoritative.
    """

    def __init__(self, polys, hashes: SketchHashes, params: SketchParams, n_rows: int, n_cols: int):
        self.hashes = hashes
        self.params = params
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self._tables: dict = {}
        self._host = None
        self._dev = None
        self.polys = polys

    # polys: numpy view of the sketch -------------------------------------------------
    @property
    def polys(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.detach().cpu().numpy()
        return self._host

    @polys.setter
    def polys(self, value) -> None:
        try:
            import torch
        except ImportError:  # pragma: no cover
            torch = None
        if torch is not None and isinstance(value, torch.Tensor) and value.is_cuda:
            self._dev = value.to(torch.float64).contiguous()
            self._host = None
        else:
            self._host = np.ascontiguousarray(value, dtype=np.float64)
            self._dev = None

    def polys_device(self, device=None):
        """(d, b) float64 CUDA tensor of the sketch."""
        import torch

        from . import _device

        dev = _device.require_cuda(device if device is not None else (self._dev.device if self._dev is not None else None))
        if self._host is not None:
            # host copy is authoritative (it may have been edited)
            return torch.from_numpy(self._host).to(dev)
        return self._dev if self._dev.device == dev else self._dev.to(dev)

    @property
    def words(self) -> np.ndarray:
        return self.hashes.packed_words()

    @property
    def is_square(self) -> bool:
        return self.n_rows == self.n_cols == self.params.n

    def table(self, which: str) -> np.ndarray:
        """Cached bucket/sign tables (sketch.py:139-149), computed on the GPU."""
        cached = self._tables.get(which)
        if cached is None:
            n = self.n_rows if which in ("h1", "s1") else self.n_cols
            cached = self.hashes.bucket_table(which, n) if which.startswith("h") else self.hashes.sign_table(which, n)
            self._tables[which] = cached
        return cached

    def __eq__(self, other) -> bool:  # dataclass-like equality on the observable state
        if not isinstance(other, ProductSketch):
            return NotImplemented
        return (self.params == other.params and self.hashes == other.hashes and self.n_rows == other.n_rows
                and self.n_cols == other.n_cols and np.array_equal(self.polys, other.polys))

    def __repr__(self) -> str:
        return (f"ProductSketch(params={self.params!r}, n_rows={self.n_rows}, n_cols={self.n_cols}, "
                f"hashes={self.hashes.digest()})")


# ----------------------------------------------------------------------------- compress
def _as_matrix(m, what: str, device):
    from . import _device

    if hasattr(m, "ndim") and m.ndim != 2:
        raise InvalidParameterError(f"{what} must be a 2-D array")
    if not hasattr(m, "ndim"):
        arr = np.asarray(m, dtype=np.float64)
        if arr.ndim != 2:
            raise InvalidParameterError(f"{what} must be a 2-D array")
        m = arr
    return _device.as_f64(m, device)


def _shape(m):
    return tuple(int(s) for s in (m.shape if hasattr(m, "shape") else np.asarray(m).shape))


def _check_2d(m, what: str):
    shp = _shape(m)
    if len(shp) != 2:
        raise InvalidParameterError(f"{what} must be a 2-D array")
    return shp


@functools.lru_cache(maxsize=256)
def _drawn(seed: int, d: int, b: int):
    """The sketch's hash functions and their packed words for (seed, d, b).

    The draw is a pure function of the seed (``default_rng(seed)``, the reference's
    order, hashing.py:78-132), and ``SketchHashes`` is immutable, so repeated
    compress calls with the same parameters reuse it: the numpy draw costs ~170 us of
    host time per call, which small sketches (cfg1: ~0.3 ms of device work) would
    otherwise spend with the GPU idle.
    """
    hashes = SketchHashes.draw(np.random.default_rng(seed), d, b)
    words = hashes.packed_words()
    words.setflags(write=False)
    return hashes, words


def _run(a, b, params: SketchParams, threads, a_layout: int, b_layout: int = 0) -> ProductSketch:
    """Steps 1-4 on device-resident operands (the reference's _run_kernel, sketch.py:238-260).

    ``a`` is A (k-minor, the reference's ``a``) or A^T (k-major, its ``at``); ``b``
    is B (k-major).  The library picks the kernel and transposes only what that
    kernel needs (the reference always copies A.T, sketch.py:305-307).
    """
    from . import _device

    m_a = a.shape[1] if a_layout == _device.KMINOR else a.shape[0]
    if m_a != b.shape[0]:
        raise InvalidParameterError(f"inner dimensions must match, got {m_a} and {b.shape[0]}")
    effective_threads(threads)
    hashes, words = _drawn(int(params.seed), params.d, params.b)
    _check_depth(params)
    acc = _device.compress_accumulate(a, b, words, params.d, params.log2b, params.transform, 0, m_a,
                                      a_layout=a_layout, b_layout=b_layout)
    polys = _device.finalize(acc, params.d, params.log2b, params.transform)
    n_rows = a.shape[0] if a_layout == _device.KMINOR else a.shape[1]
    return ProductSketch(polys=polys, hashes=hashes, params=params, n_rows=n_rows, n_cols=b.shape[1])


def _is_host(m) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(m, torch.Tensor):
        return not m.is_cuda
    return True  # numpy arrays and nested sequences live on the host


def _run_host(a, b, params: SketchParams, threads, a_layout: int, dev) -> ProductSketch:
    """_run for host-resident operands: k-slabs are uploaded while earlier slabs
    compute (pinned host tensors give the full PCIe rate)."""
    from . import _device

    a = _device.host_f64(a)
    b = _device.host_f64(b)
    effective_threads(threads)
    hashes, words = _drawn(int(params.seed), params.d, params.b)
    _check_depth(params)
    acc = _device.compress_host(a, b, words, params.d, params.log2b, params.transform, a_layout, dev)
    polys = _device.finalize(acc, params.d, params.log2b, params.transform)
    n_rows = a.shape[0] if a_layout == _device.KMINOR else a.shape[1]
    return ProductSketch(polys=polys, hashes=hashes, params=params, n_rows=n_rows, n_cols=b.shape[1])


def _dispatch(a, b, params, threads, a_layout, dev, what_a):
    if _is_host(a) and _is_host(b):
        return _run_host(a, b, params, threads, a_layout, dev)
    return _run(_as_matrix(a, what_a, dev), _as_matrix(b, "right operand", dev), params, threads, a_layout)


def _check_depth(params: SketchParams) -> None:
    # any odd d as the reference (sketch.py:75-76), up to the device path's limit; past
    # 63 repetitions the kernels run in groups of 63 and extraction reads the hashes
    # from device memory
    from ._lib import MAX_DEPTH_TOTAL

    if params.d > MAX_DEPTH_TOTAL:
        raise InvalidParameterError(f"d={params.d} exceeds the device path's maximum depth {MAX_DEPTH_TOTAL}")


def compress(a, b, params: SketchParams, threads: int | None = None, device=None) -> ProductSketch:
    """Sketch the product of square n x n operands (sketch.py:289-302)."""
    from . import _device

    sa = _check_2d(a, "left operand")
    sb = _check_2d(b, "right operand")
    n = params.n
    if sa != (n, n) or sb != (n, n):
        raise InvalidParameterError(f"operands must both be {n} x {n}, got {sa} and {sb}")
    effective_threads(threads)
    dev = _device.require_cuda(device)
    return _dispatch(a, b, params, threads, _device.KMINOR, dev, "left operand")


def compress_pretransposed(at, b, params: SketchParams, threads: int | None = None, device=None) -> ProductSketch:
    """Like ``compress`` with A given transposed (sketch.py:310-321)."""
    from . import _device

    sa = _check_2d(at, "left operand (transposed)")
    sb = _check_2d(b, "right operand")
    n = params.n
    if sa != (n, n) or sb != (n, n):
        raise InvalidParameterError(f"operands must both be {n} x {n}, got {sa} and {sb}")
    effective_threads(threads)
    dev = _device.require_cuda(device)
    return _dispatch(at, b, params, threads, _device.KMAJOR, dev, "left operand (transposed)")


def compress_rect(a, b, params: SketchParams, threads: int | None = None, device=None) -> ProductSketch:
    """Sketch a rectangular product A (n1 x m) @ B (m x n2), m = params.n (sketch.py:324-340)."""
    from . import _device

    sa = _check_2d(a, "left operand")
    sb = _check_2d(b, "right operand")
    if sa[1] != params.n or sb[0] != params.n:
        raise InvalidParameterError(f"inner dimension must equal params.n={params.n}, got {sa} x {sb}")
    effective_threads(threads)
    dev = _device.require_cuda(device)
    return _dispatch(a, b, params, threads, _device.KMINOR, dev, "left operand")


def compress_seeds(a, b, params: SketchParams, seeds, threads: int | None = None, device=None) -> list:
    """Independent sketches of one product for many hash seeds, batched.

    The reference's Monte-Carlo drivers (variance_experiment / correctness_run,
    experiments.py:216-312) call ``compress`` once per seed.  Here the seeds'
    repetitions are stacked into one deeper sketch (up to 63 repetitions per
    launch), so each operand slab is read once for all of them; every repetition
    is computed exactly as in its own ``compress`` call, so sketch ``s`` equals
    ``compress(a, b, replace(params, seed=seeds[s]))``.
    """
    from dataclasses import replace

    from . import _device
    from ._lib import MAX_DEPTH

    seeds = [int(x) for x in seeds]
    sa = _check_2d(a, "left operand")
    sb = _check_2d(b, "right operand")
    n = params.n
    if sa != (n, n) or sb != (n, n):
        raise InvalidParameterError(f"operands must both be {n} x {n}, got {sa} and {sb}")
    per = [replace(params, seed=s) for s in seeds]  # validates every seed
    effective_threads(threads)
    dev = _device.require_cuda(device)
    host = _is_host(a) and _is_host(b)
    if host:
        a_op, b_op = _device.host_f64(a), _device.host_f64(b)
    else:
        a_op, b_op = _as_matrix(a, "left operand", dev), _as_matrix(b, "right operand", dev)
    d = params.d
    # seeds stacked into one launch of the kernel family a single-seed compress would use,
    # so every sketch is bit-identical to its own compress call
    single = _device.compress_kernel(params.transform, d, params.log2b, n, n, n)
    group = max(1, MAX_DEPTH // d)
    while group > 1 and _device.compress_kernel(params.transform, d * group, params.log2b, n, n, n) != single:
        group -= 1
    out = []
    for g0 in range(0, len(per), group):
        ps = per[g0:g0 + group]
        hs = [_drawn(int(p.seed), d, p.b)[0] for p in ps]
        stacked = SketchHashes(h1=sum((h.h1 for h in hs), ()), h2=sum((h.h2 for h in hs), ()),
                               s1=sum((h.s1 for h in hs), ()), s2=sum((h.s2 for h in hs), ()))
        words = stacked.packed_words()
        D = d * len(ps)
        if host:
            acc = _device.compress_host(a_op, b_op, words, D, params.log2b, params.transform, _device.KMINOR, dev)
        else:
            acc = _device.compress_accumulate(a_op, b_op, words, D, params.log2b, params.transform, 0, n,
                                              a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
        polys = _device.finalize(acc, D, params.log2b, params.transform)
        for q, (p, h) in enumerate(zip(ps, hs)):
            out.append(ProductSketch(polys=polys[q * d:(q + 1) * d].clone(), hashes=h, params=p, n_rows=n, n_cols=n))
    return out


# ----------------------------------------------------------------------------- decompress
def combine_index(sketch: ProductSketch, k1: int, k2: int) -> int:
    """XOR for fwht, addition mod b for fft (sketch.py:343-347)."""
    if sketch.params.transform == "fwht":
        return k1 ^ k2
    return (k1 + k2) % sketch.params.b


def sketch_estimates(sketch: ProductSketch, i: int, j: int) -> np.ndarray:
    """The d per-repetition estimates of entry (i, j) (sketch.py:350-367)."""
    if not (0 <= i < sketch.n_rows and 0 <= j < sketch.n_cols):
        raise InvalidParameterError(f"entry ({i}, {j}) outside {sketch.n_rows} x {sketch.n_cols}")
    h = sketch.hashes
    polys = sketch.polys
    out = np.empty(h.d)
    for t in range(h.d):
        idx = combine_index(sketch, eval_bucket(h.h1[t], i), eval_bucket(h.h2[t], j))
        out[t] = eval_sign(h.s1[t], i) * eval_sign(h.s2[t], j) * polys[t, idx]
    return out


def decompress_entry(sketch: ProductSketch, i: int, j: int) -> float:
    """Median-of-sketches estimate of entry (i, j) (sketch.py:370-372)."""
    return float(np.median(sketch_estimates(sketch, i, j)))


def decompress_entries(sketch: ProductSketch, ij, *, with_estimates: bool = False, device=None,
                       as_numpy: bool = True):
    """Batched per-entry queries on the device-resident sketch: the median estimate
    of every (i, j) pair in ``ij`` (shape (q, 2)), equal to ``decompress_entry`` per
    pair; with ``with_estimates`` also the (q, d) per-repetition values of
    ``sketch_estimates`` (sketch.py:350-372)."""
    import torch

    from . import _device

    arr = ij if isinstance(ij, torch.Tensor) else torch.as_tensor(np.asarray(ij, dtype=np.int64))
    if arr.ndim != 2 or arr.shape[1] != 2:
        raise InvalidParameterError("ij must have shape (q, 2)")
    if arr.numel():
        lo = arr.min(dim=0).values.tolist()
        hi = arr.max(dim=0).values.tolist()
        if lo[0] < 0 or lo[1] < 0 or hi[0] >= sketch.n_rows or hi[1] >= sketch.n_cols:
            raise InvalidParameterError(f"entries outside {sketch.n_rows} x {sketch.n_cols}")
    p = sketch.params
    polys = sketch.polys_device(device)
    est, reps = _device.query(polys, sketch.words, p.d, p.log2b, p.transform, sketch.n_rows, sketch.n_cols, arr,
                              want_reps=with_estimates)
    if as_numpy:
        est = est.cpu().numpy()
        reps = reps.cpu().numpy() if reps is not None else None
    return (est, reps) if with_estimates else est


def decompress_rows(sketch: ProductSketch, r0: int = 0, r1: int | None = None, *, device=None, out=None):
    """Estimates of output rows [r0, r1) as a CUDA tensor (the row-sharded unit)."""
    from . import _device

    r1 = sketch.n_rows if r1 is None else r1
    if not (0 <= r0 <= r1 <= sketch.n_rows):
        raise InvalidParameterError(f"row range [{r0}, {r1}) outside {sketch.n_rows} rows")
    p = sketch.params
    polys = sketch.polys_device(device)
    est, _, _ = _device.extract(polys, sketch.words, p.d, p.log2b, p.transform, sketch.n_rows, sketch.n_cols,
                                r0, r1, want_est=True, est_out=out)
    return est


def decompress_all(sketch: ProductSketch, *, device=None, out=None, as_numpy: bool = True):
    """Estimates for every entry (sketch.py:375-399); bit-identical to the
    per-entry path.  Returns numpy by default (reference behaviour); pass
    ``as_numpy=False`` to keep the CUDA tensor, or ``out`` (numpy or a pinned
    host tensor) to receive the copy."""
    est = decompress_rows(sketch, 0, sketch.n_rows, device=device)
    if out is not None:
        import torch

        if isinstance(out, torch.Tensor):
            out.copy_(est, non_blocking=False)
        else:
            out[...] = est.cpu().numpy()
        return out
    return est.cpu().numpy() if as_numpy else est


def heavy_hitters(sketch: ProductSketch, threshold: float = 0.5, strict: bool = True, *, r0: int = 0,
                  r1: int | None = None, device=None, with_estimates: bool = False, as_numpy: bool = True):
    """Entries whose median estimate clears the threshold, in row-major order.

    ``strict`` selects |est| > threshold (BASELINE cfg5); ``strict=False`` is the
    inclusive comparator of experiments.py:164 (|est| >= 0.5).  The reference has
    no standalone API for this; it is fused into the extraction kernel here.
    Returns an (k, 2) int64 array of (i, j) pairs (and the estimate rows if asked).
    """
    from . import _device

    r1 = sketch.n_rows if r1 is None else r1
    if not (0 <= r0 <= r1 <= sketch.n_rows):
        raise InvalidParameterError(f"row range [{r0}, {r1}) outside {sketch.n_rows} rows")
    p = sketch.params
    polys = sketch.polys_device(device)
    est, _, pairs = _device.extract(polys, sketch.words, p.d, p.log2b, p.transform, sketch.n_rows, sketch.n_cols,
                                    r0, r1, want_est=with_estimates, thr=threshold, strict=strict, want_pairs=True)
    if as_numpy:
        pairs = pairs.cpu().numpy()
        est = est.cpu().numpy() if est is not None else None
    return (pairs, est) if with_estimates else pairs


def extract_all(sketch: ProductSketch, threshold: float = 0.5, strict: bool = True, *, r0: int = 0,
                r1: int | None = None, device=None, est_out=None):
    """Step 5 in one pass: the estimate rows [r0, r1) and their heavy-hitter pairs
    (CUDA tensors).  This is ``decompress_all`` fused with the threshold.  With a
    host ``est_out`` the rows are streamed out in blocks and the pairs come back as
    a pinned host tensor; both are complete on return."""
    from . import _device

    r1 = sketch.n_rows if r1 is None else r1
    if not (0 <= r0 <= r1 <= sketch.n_rows):
        raise InvalidParameterError(f"row range [{r0}, {r1}) outside {sketch.n_rows} rows")
    p = sketch.params
    polys = sketch.polys_device(device)
    if est_out is not None and not est_out.is_cuda:
        # host destination (pinned for full speed): extraction of row block q+1 overlaps the copy-out of q
        pairs = _device.extract_host(polys, sketch.words, p.d, p.log2b, p.transform, sketch.n_rows, sketch.n_cols,
                                     r0, r1, threshold, strict, est_out)
        return est_out, pairs
    est, _, pairs = _device.extract(polys, sketch.words, p.d, p.log2b, p.transform, sketch.n_rows, sketch.n_cols,
                                    r0, r1, want_est=True, thr=threshold, strict=strict, want_pairs=True,
                                    est_out=est_out)
    return est, pairs


def estimate_workspace_bytes(n: int, b: int, d: int, transform: str, threads: int) -> int:
    """Host-memory estimate of the reference path (sketch.py:402-417), kept for API parity."""
    f8, c16 = 8, 16
    half = b // 2 + 1
    operands = 3 * n * n * f8
    tables = 4 * d * n * f8
    if transform == "fwht":
        kernel = (threads + 1) * d * b * f8 + threads * (d + 1) * b * f8
    else:
        kernel = 2 * (threads + 1) * d * half * c16 + threads * b * c16 + d * b * f8
    block = max(1, (1 << 24) // max(1, d * n))
    decomp = n * n * f8 + 3 * d * block * n * f8
    return operands + tables + kernel + decomp


def device_workspace_bytes(n1: int, n2: int, m: int, params: SketchParams) -> int:
    """Device bytes the compress call needs beyond its operands and outputs."""
    import ctypes

    from . import _lib

    lib = _lib.load()
    out = ctypes.c_int64(0)
    _lib.check(lib.smm_compress_workspace(_lib.VARIANT[params.transform], params.d, params.log2b, n1, n2, 0, m,
                                          ctypes.byref(out)))
    return int(out.value)


# ----------------------------------------------------------------------------- container
def sketch_to_bytes(sketch: ProductSketch) -> bytes:
    """Serialize a square sketch: header, 8d hash words, d*b float64 (sketch.py:420-436)."""
    if not sketch.is_square:
        raise InvalidParameterError("only square sketches can be serialized")
    p = sketch.params
    header = SKETCH_HEADER.pack(SKETCH_MAGIC, SKETCH_VERSION, p.n, p.b, p.d, TRANSFORM_CODES[p.transform], p.seed)
    return header + sketch.words.astype("<u8").tobytes() + sketch.polys.astype("<f8").tobytes(order="C")


def sketch_from_bytes(buf: bytes) -> ProductSketch:
    """Parse a .skch container (sketch.py:439-482)."""
    if len(buf) < SKETCH_HEADER.size:
        raise FormatError("sketch container truncated before header")
    magic, version, n, b, d, tcode, seed = SKETCH_HEADER.unpack_from(buf)
    if magic != SKETCH_MAGIC:
        raise FormatError(f"bad sketch magic {magic!r}")
    if version != SKETCH_VERSION:
        raise FormatError(f"unsupported sketch container version {version}")
    if tcode not in TRANSFORM_NAMES:
        raise FormatError(f"unknown transform code {tcode}")
    try:
        params = SketchParams(n=int(n), b=int(b), d=int(d), transform=TRANSFORM_NAMES[tcode], seed=int(seed))
    except InvalidParameterError as exc:
        raise FormatError(f"invalid sketch header: {exc}") from exc
    off = SKETCH_HEADER.size
    payload = off + 8 * 8 * params.d
    want = payload + 8 * params.d * params.b
    if len(buf) != want:
        raise FormatError(f"sketch payload has {len(buf)} bytes, expected {want}")
    words = np.frombuffer(buf, dtype="<u8", count=8 * params.d, offset=off)
    hashes = SketchHashes.from_words(words, params.d, params.b)
    polys = np.frombuffer(buf, dtype="<f8", offset=payload).reshape(params.d, params.b).astype(np.float64)
    return ProductSketch(polys=polys, hashes=hashes, params=params, n_rows=params.n, n_cols=params.n)


def save_sketch(path, sketch: ProductSketch) -> None:
    Path(path).write_bytes(sketch_to_bytes(sketch))


def load_sketch(path) -> ProductSketch:
    return sketch_from_bytes(Path(path).read_bytes())


__all__ = [
    "HashPair", "ProductSketch", "SketchParams", "TRANSFORMS", "combine_index", "compress", "compress_pretransposed",
    "compress_rect", "decompress_all", "decompress_entry", "decompress_rows", "derive_params", "extract_all",
    "device_workspace_bytes", "effective_threads", "estimate_workspace_bytes", "heavy_hitters", "load_sketch",
    "save_sketch", "sketch_estimates", "sketch_from_bytes", "sketch_to_bytes", "check_buckets",
]
