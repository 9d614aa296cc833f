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
    with torch.cuda.device(x.device):
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
                        b_layout: int = KMAJOR, accumulate: bool = False) -> torch.Tensor:
    """Pre-inverse accumulator of inner indices [k0, k1).

    ``a`` is A^T (KMAJOR, rows = k) or A itself (KMINOR, columns = k); ``b`` is B
    (KMAJOR) or B^T (KMINOR).  Views with a row stride are used in place.
    ``accumulate`` adds to ``acc`` instead of overwriting it (SMM_FLAG_ACCUMULATE).
    """
    lib = _lib.load()
    a = _rowmajor(a)
    b = _rowmajor(b)
    dev = a.device
    n1 = a.shape[1] if a_layout == KMAJOR else a.shape[0]
    n2 = b.shape[1] if b_layout == KMAJOR else b.shape[0]
    v = _lib.VARIANT[variant]
    if accumulate:
        if acc is None:
            raise InvalidParameterError("accumulate=True needs an accumulator to add to")
        v |= _lib.FLAG_ACCUMULATE
    nbytes = ctypes.c_int64(0)
    _lib.check(lib.smm_compress_workspace_ex(v, d, log2b, n1, n2, k0, k1, a_layout, b_layout, ctypes.byref(nbytes)))
    # the library launches on the current device: make it the operands' device
    with torch.cuda.device(dev):
        ws = workspace(nbytes.value, dev)
        if acc is None:
            acc = torch.empty(acc_shape(variant, d, 1 << log2b), dtype=torch.float64, device=dev)
        words, wp = words_ptr(words)
        _lib.check(lib.smm_compress_accumulate_ex(v, ptr(a), a.stride(0), a_layout, ptr(b), b.stride(0), b_layout,
                                                  n1, n2, k0, k1, wp, d, log2b, ptr(acc), ptr(ws), ws.numel(),
                                                  stream_ptr(dev)))
    return acc


def compress_kernel(variant: str, d: int, log2b: int, n1: int, n2: int, m: int) -> int:
    """The compress kernel family (SMM_KERNEL_*) the library picks for these shapes."""
    lib = _lib.load()
    out = ctypes.c_int(-1)
    _lib.check(lib.smm_compress_kernel(_lib.VARIANT[variant], d, log2b, n1, n2, 0, m, ctypes.byref(out)))
    return int(out.value)


def copy2d(dst: torch.Tensor, src: torch.Tensor, stream: torch.cuda.Stream) -> None:
    """dst[...] = src for 2-D row-strided views (host or device, any direction) on ``stream``."""
    lib = _lib.load()
    if dst.shape != src.shape or dst.dtype != src.dtype or dst.stride(1) != 1 or src.stride(1) != 1:
        raise InvalidParameterError("copy2d needs equal-shape row-strided views")
    es = src.element_size()
    _lib.check(lib.smm_copy2d(ptr(dst), dst.stride(0) * es, ptr(src), src.stride(0) * es, src.shape[1] * es,
                              src.shape[0], ctypes.c_void_p(stream.cuda_stream)))


def host_f64(x) -> torch.Tensor:
    """A host operand as a row-strided float64 CPU tensor (no copy when it already is one)."""
    if isinstance(x, torch.Tensor):
        t = x if x.dtype == torch.float64 else x.to(torch.float64)
    else:
        t = torch.from_numpy(np.asarray(x, dtype=np.float64))
    if t.dim() != 2:
        raise InvalidParameterError("operands must be 2-D")
    if t.stride(1) != 1:
        t = t.contiguous()
    return t


def stream_chunk(m: int, n_max: int) -> int:
    """k-slab width for host-streamed compress: ~8 slabs, a multiple of 32 (k-tile aligned)."""
    kc = max(256, -(-m // 8))
    kc = -(-kc // 32) * 32
    # keep one slab of both operands under ~1 GiB
    while kc > 256 and 8 * kc * n_max * 2 > (1 << 30):
        kc //= 2
    return max(32, min(kc, -(-m // 32) * 32))


def _slab_bounds(m: int, kc: int) -> list:
    """k-slabs of width kc, the last one split geometrically (kc/2, kc/4, kc/8, kc/8;
    multiples of 32): uploads outpace nothing, so after the final upload only the last
    piece's compute remains exposed — keep it small."""
    bounds = [(c0, min(m, c0 + kc)) for c0 in range(0, m, kc)]
    c0, c1 = bounds[-1]
    w = c1 - c0
    if len(bounds) > 1 and w >= 128:
        cuts = [c0]
        for frac in (2, 4, 8):
            step = ((w // frac + 31) // 32) * 32
            if cuts[-1] + step < c1:
                cuts.append(cuts[-1] + step)
        cuts.append(c1)
        bounds = bounds[:-1] + [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    return bounds


def compress_host(a: torch.Tensor, b: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str,
                  a_layout: int, device: torch.device, chunk: int | None = None) -> torch.Tensor:
    """Pre-inverse accumulator of host-resident operands, streamed in k-slabs.

    Slab c+1 is uploaded on a copy stream (2-D copies: a k-slab of a row-major A is
    a column block) while the kernel accumulates slab c; every slab after the first
    is added in SMM_FLAG_ACCUMULATE mode, so with the two-pass FWHT kernel the
    result is bit-identical to one call over the whole inner range.
    """
    m = a.shape[1] if a_layout == KMINOR else a.shape[0]
    n1 = a.shape[0] if a_layout == KMINOR else a.shape[1]
    n2 = b.shape[1]
    if b.shape[0] != m:
        raise InvalidParameterError(f"inner dimensions must match, got {m} and {b.shape[0]}")
    kc = chunk or stream_chunk(m, max(n1, n2))
    acc = torch.empty(acc_shape(variant, d, 1 << log2b), dtype=torch.float64, device=device)
    if m == 0:
        return compress_accumulate(torch.empty((0, n1) if a_layout == KMAJOR else (n1, 0), dtype=torch.float64,
                                               device=device), torch.empty((0, n2), dtype=torch.float64, device=device),
                                   words, d, log2b, variant, 0, 0, acc, a_layout, KMAJOR)
    with torch.cuda.device(device):
        return _compress_host(a, b, words, d, log2b, variant, a_layout, device, kc, acc, m, n1, n2)


def _compress_host(a, b, words, d, log2b, variant, a_layout, device, kc, acc, m, n1, n2):
    compute = torch.cuda.current_stream(device)
    copy = torch.cuda.Stream(device)
    abuf = [torch.empty((n1, kc) if a_layout == KMINOR else (kc, n1), dtype=torch.float64, device=device)
            for _ in range(2)]
    bbuf = [torch.empty((kc, n2), dtype=torch.float64, device=device) for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    slabs = _slab_bounds(m, kc)

    def upload(c):
        c0, c1 = slabs[c]
        w = c1 - c0
        q = c % 2
        with torch.cuda.stream(copy):
            if c >= 2:
                copy.wait_event(freed[q])
            if a_layout == KMINOR:
                copy2d(abuf[q][:, :w], a[:, c0:c1], copy)
            else:
                copy2d(abuf[q][:w], a[c0:c1], copy)
            copy2d(bbuf[q][:w], b[c0:c1], copy)
            loaded[q].record(copy)

    # the ring buffers come from the compute stream's pool: blocks freed there may still
    # be in use by queued kernels, so the copy stream starts behind the compute stream
    copy.wait_stream(compute)
    upload(0)
    for c, (c0, c1) in enumerate(slabs):
        if c + 1 < len(slabs):
            upload(c + 1)
        q = c % 2
        w = c1 - c0
        compute.wait_event(loaded[q])
        av = abuf[q][:, :w] if a_layout == KMINOR else abuf[q][:w]
        compress_accumulate(av, bbuf[q][:w], words, d, log2b, variant, 0, w, acc, a_layout, KMAJOR,
                            accumulate=c > 0)
        freed[q].record(compute)
    compute.wait_stream(copy)
    # the DMA reads the caller's host tensors asynchronously (pinned memory): return only
    # once the last upload has finished, so the caller may free or reuse them
    uploaded = torch.cuda.Event()
    uploaded.record(copy)
    uploaded.synchronize()
    return acc


def kernel_timing(enable: bool) -> None:
    """Bracket every compress / extraction kernel launch with CUDA events (bench evidence)."""
    _lib.check(_lib.load().smm_kernel_timing(1 if enable else 0))


def kernel_timing_read(channel: int) -> tuple[float, int]:
    """(summed device ms, launches) recorded on channel 0 (compress) or 1 (extraction); clears them."""
    tot = ctypes.c_double(0.0)
    cnt = ctypes.c_int64(0)
    _lib.check(_lib.load().smm_kernel_timing_read(channel, ctypes.byref(tot), ctypes.byref(cnt)))
    return float(tot.value), int(cnt.value)


def finalize(acc: torch.Tensor, d: int, log2b: int, variant: str) -> torch.Tensor:
    lib = _lib.load()
    polys = torch.empty((d, 1 << log2b), dtype=torch.float64, device=acc.device)
    with torch.cuda.device(acc.device):
        _lib.check(lib.smm_finalize(_lib.VARIANT[variant], ptr(acc), ptr(polys), d, log2b, stream_ptr(acc.device)))
    return polys


def pair_capacity(rows: int, n2: int) -> int:
    """Heavy-hitter pair buffer written without knowing the count (1/8 of the grid,
    at least 64K pairs); a larger count is re-emitted from the kept bitmask."""
    return int(min(rows * n2, max(1 << 16, (rows * n2) // 8)))


class PendingPairs:
    """Heavy-hitter pairs of one extract call, written on the device up to a capacity;
    ``resolve()`` reads the device count (the call's only host sync) and re-emits
    the list from the call's bitmask in the rare case it overflowed."""

    def __init__(self, count, buf, ws, n2, r0, r1, dev):
        self.count, self.buf, self.ws, self.n2, self.r0, self.r1, self.dev = count, buf, ws, n2, r0, r1, dev

    def resolve(self, cnt: int | None = None) -> torch.Tensor:
        cnt = int(self.count.item()) if cnt is None else cnt
        if cnt > self.buf.shape[0]:
            lib = _lib.load()
            self.buf = torch.empty((cnt, 2), dtype=torch.int64, device=self.dev)
            with torch.cuda.device(self.dev):
                _lib.check(lib.smm_hh_pairs(ptr(self.ws), self.n2, self.r0, self.r1, ptr(self.buf), cnt,
                                            stream_ptr(self.dev)))
        self.ws = None
        return self.buf[:cnt]


def extract(polys: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str, n1: int, n2: int,
            r0: int = 0, r1: int | None = None, want_est: bool = True, thr: float = 0.5, strict: bool = True,
            want_pairs: bool = False, est_out: torch.Tensor | None = None, defer_pairs: bool = False):
    """Rows [r0, r1) of the estimate grid and the heavy hitters |est| >(=) thr.

    The pair list is written by the kernel that follows the extraction with no
    host round trip in between (capacity ``pair_capacity``); the count is read
    once at the end, or never with ``defer_pairs`` (then ``pairs`` is a
    ``PendingPairs`` to resolve later)."""
    lib = _lib.load()
    dev = polys.device
    r1 = n1 if r1 is None else r1
    rows = r1 - r0
    with torch.cuda.device(dev):
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
        cap = pair_capacity(rows, n2) if want_pairs else 0
        buf = torch.empty((cap, 2), dtype=torch.int64, device=dev) if want_pairs else None
        _lib.check(lib.smm_extract(v, ptr(polys), wp, d, log2b, n1, n2, r0, r1, ptr(est), ld, float(thr),
                                   1 if strict else 0, ptr(buf), cap, ptr(count), ptr(ws), ws.numel(),
                                   stream_ptr(dev)))
    pairs = None
    if want_pairs:
        pairs = PendingPairs(count, buf, ws, n2, r0, r1, dev)
        if not defer_pairs:
            pairs = pairs.resolve()
    return est, count, pairs


def query(polys: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str, n1: int, n2: int,
          ij: torch.Tensor, want_reps: bool = False):
    """Median estimates (and optionally the d per-repetition values) at int64 (i, j) pairs."""
    lib = _lib.load()
    dev = polys.device
    ij = ij.to(device=dev, dtype=torch.int64).contiguous()
    count = ij.shape[0]
    est = torch.empty(count, dtype=torch.float64, device=dev)
    reps = torch.empty((count, d), dtype=torch.float64, device=dev) if want_reps else None
    words, wp = words_ptr(words)
    with torch.cuda.device(dev):
        _lib.check(lib.smm_query(_lib.VARIANT[variant], ptr(polys), wp, d, log2b, n1, n2, ptr(ij), count, ptr(est),
                                 ptr(reps), stream_ptr(dev)))
    return est, reps


def extract_host(polys: torch.Tensor, words: np.ndarray, d: int, log2b: int, variant: str, n1: int, n2: int,
                 r0: int, r1: int, thr: float, strict: bool, est_host: torch.Tensor, block_rows: int | None = None):
    """Rows [r0, r1) of the estimates into a host tensor, in row blocks: block q+1
    is extracted while block q is copied out on a copy stream (2-slot device ring).
    Returns the heavy-hitter pairs as a pinned host tensor; both are complete on return."""
    dev = polys.device
    rows = r1 - r0
    if tuple(est_host.shape) != (rows, n2) or est_host.dtype != torch.float64 or est_host.stride(1) != 1:
        raise InvalidParameterError(f"est_out must be a ({rows}, {n2}) float64 row-major tensor")
    if rows == 0 or n2 == 0:
        _, _, pairs = extract(polys, words, d, log2b, variant, n1, n2, r0, r1, want_est=False, thr=thr,
                              strict=strict, want_pairs=True)
        return pairs.cpu()
    R = block_rows or max(1, min(rows, (128 << 20) // (8 * n2)))
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    ring = [torch.empty((R, n2), dtype=torch.float64, device=dev) for _ in range(min(2, -(-rows // R)))]
    ready = [torch.cuda.Event() for _ in ring]
    done = [torch.cuda.Event() for _ in ring]
    pending = []
    with torch.cuda.device(dev):
        copy.wait_stream(compute)  # ring blocks may reuse memory still in use on the compute stream
        for bi, q0 in enumerate(range(r0, r1, R)):
            q1 = min(r1, q0 + R)
            slot = bi % len(ring)
            if bi >= len(ring):
                compute.wait_event(done[slot])
            _, _, pr = extract(polys, words, d, log2b, variant, n1, n2, q0, q1, want_est=True, thr=thr,
                               strict=strict, want_pairs=True, est_out=ring[slot][:q1 - q0], defer_pairs=True)
            pending.append(pr)
            ready[slot].record(compute)
            with torch.cuda.stream(copy):
                copy.wait_event(ready[slot])
                copy2d(est_host[q0 - r0:q1 - r0], ring[slot][:q1 - q0], copy)
                done[slot].record(copy)
        # no host round trip per block: every block's count is read once, after all are queued
        counts = torch.cat([pr.count for pr in pending]).cpu().tolist()
        pairs = [pr.resolve(c) for pr, c in zip(pending, counts)]
        pairs = torch.cat(pairs) if len(pairs) > 1 else pairs[0]
        pairs_host = torch.empty(pairs.shape, dtype=pairs.dtype, pin_memory=True)
        pairs_host.copy_(pairs, non_blocking=True)  # on the compute stream, behind the last extraction
        compute.wait_stream(copy)
        compute.synchronize()  # the reference's decompress_all is synchronous: est_host is complete
    return pairs_host


def fwht_batched(x: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
    lib = _lib.load()
    n = x.shape[-1]
    log2n = n.bit_length() - 1
    batch = x.numel() // n if n else 0
    with torch.cuda.device(x.device):
        _lib.check(lib.smm_fwht_batched(ptr(x), batch, log2n, float(scale), stream_ptr(x.device)))
    return x


def fft_batched(z: torch.Tensor, inverse: bool = False, scale: float = 1.0) -> torch.Tensor:
    """z: complex128 CUDA tensor (..., n), transformed in place."""
    lib = _lib.load()
    n = z.shape[-1]
    log2n = n.bit_length() - 1
    batch = z.numel() // n if n else 0
    with torch.cuda.device(z.device):
        _lib.check(lib.smm_fft_batched(ptr(z), batch, log2n, 1 if inverse else 0, float(scale),
                                       stream_ptr(z.device)))
    return z
