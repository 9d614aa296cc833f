"""CPU ORACLE for the sketched-product hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the CPU baseline — never as the thing measured or shipped.  The product
package ``paper_2601_09477_b200`` never imports it.

It restates the reference ``sketchmm`` algorithm (paths relative to
/root/reference/pkg/src/sketchmm):

* hash drawing: ``draw_hash`` hashing.py:78-85, ``SketchHashes.draw``
  hashing.py:123-132 (numpy PCG64 stream, order h1, h2, s1, s2; (a, c) per
  function); ``packed_words`` hashing.py:146-152.
* tables: ``bucket_many``/``sign_many`` hashing.py:64-75 and
  ``bucket_table``/``sign_table`` hashing.py:134-144.
* FFT tables: ``fft_tables`` transforms.py:80-97 (numpy, identical calls).
* compress kernels + chunking: sketch.py:117-120, 152-260 — in C
  (oracle/csrc/sketch_oracle.c), bit-identical to the reference at the same
  chunk count (pinned by tests/test_oracle_pins.py).
* ``compress_slow``: the slow per-outer-product oracle of the reference test
  suite (tests/helpers.py:49-71), pure numpy, tiny sizes only.
* ``decompress``: sketch.py:375-399 plus the heavy-hitter comparator of
  experiments.py:136-168 (inclusive) or BASELINE cfg5 (strict).

Parity pin: every function here is checked against golden vectors produced by
running the reference itself (tools/make_golden.py -> tests/golden/).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libsketch_oracle.so"
_lib = None

MASK64 = (1 << 64) - 1


def build() -> Path:
    """Compile the C restatement (idempotent)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        D = ctypes.c_double
        lib.oracle_compress_fwht.argtypes = [P, P, I64, I64, I64, P, P, P, P, I, I64, P, P, I, I, P]
        lib.oracle_accumulate_fwht.argtypes = [P, P, I64, I64, P, P, P, P, I, I64, I64, I64, I, P]
        lib.oracle_compress_fft.argtypes = [P, P, I64, I64, I64, P, P, P, P, I, I64, P, P, P, P, P, I, I, P]
        lib.oracle_decompress.argtypes = [P, I, I64, I, P, P, P, P, I64, I64, I64, I64, P, D, I, P, I64, P, I]
        lib.oracle_fwht_inplace.argtypes = [P, I64]
        lib.oracle_fft_inplace.argtypes = [P, I64, P, P]
        for f in (lib.oracle_compress_fwht, lib.oracle_accumulate_fwht, lib.oracle_compress_fft, lib.oracle_decompress):
            f.restype = I
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- hashes
def draw_words(seed: int, d: int, b: int) -> np.ndarray:
    """The 8d hash words of a depth-d, width-b sketch in draw order.

    Mirrors hashing.py:78-85/123-132: one ``default_rng(seed)``; each function
    consumes ``integers(0, 2**64, size=2, dtype=uint64)`` as (a, c); groups in
    the order h1[0..d), h2[0..d), s1[0..d), s2[0..d).
    """
    rng = np.random.default_rng(seed)
    words = []
    for _ in range(4 * d):
        a, c = (int(v) for v in rng.integers(0, 1 << 64, size=2, dtype=np.uint64))
        words.extend((a, c))
    return np.array(words, dtype=np.uint64)


def bucket_table(words: np.ndarray, d: int, b: int, group: int, n: int) -> np.ndarray:
    """(d, n) int64 buckets of keys 0..n-1 for group 0 (h1) or 1 (h2)."""
    shift = np.uint64(64 - (int(b).bit_length() - 1))
    xs = np.arange(n, dtype=np.uint64)
    out = np.empty((d, n), dtype=np.int64)
    base = group * 2 * d
    for t in range(d):
        a = np.uint64(words[base + 2 * t])
        c = np.uint64(words[base + 2 * t + 1])
        out[t] = ((a * xs + c) >> shift).astype(np.int64)
    return out


def sign_table(words: np.ndarray, d: int, group: int, n: int) -> np.ndarray:
    """(d, n) float64 signs for group 2 (s1) or 3 (s2): 1 - 2 * top bit."""
    xs = np.arange(n, dtype=np.uint64)
    out = np.empty((d, n), dtype=np.float64)
    base = group * 2 * d
    for t in range(d):
        a = np.uint64(words[base + 2 * t])
        c = np.uint64(words[base + 2 * t + 1])
        out[t] = 1.0 - 2.0 * ((a * xs + c) >> np.uint64(63)).astype(np.float64)
    return out


def tables(words: np.ndarray, d: int, b: int, n1: int, n2: int):
    return (
        bucket_table(words, d, b, 0, n1),
        sign_table(words, d, 2, n1),
        bucket_table(words, d, b, 1, n2),
        sign_table(words, d, 3, n2),
    )


def fft_tables(b: int):
    """transforms.py:80-97, same numpy calls -> identical bits."""
    bits = b.bit_length() - 1
    rev = np.zeros(b, dtype=np.int64)
    for i in range(1, b):
        rev[i] = (rev[i >> 1] >> 1) | ((i & 1) << (bits - 1))
    k = np.arange(b // 2, dtype=np.float64)
    tw = np.exp(-2j * np.pi * k / b)
    return tw, np.conj(tw), rev


def chunk_bounds(m: int, nchunks: int):
    """sketch.py:117-120."""
    edges = np.linspace(0, m, nchunks + 1).astype(np.int64)
    return edges[:-1].copy(), edges[1:].copy()


# --------------------------------------------------------------------------- compress
def compress(a, bmat, *, b: int, d: int, transform: str, seed: int, threads: int = 1,
             pretransposed: bool = False, words: np.ndarray | None = None) -> np.ndarray:
    """Polys (d, b) exactly as the reference ``compress`` / ``compress_rect``
    with ``threads`` chunks (sketch.py:289-340 -> _run_kernel 238-260)."""
    lib = _load()
    av = np.ascontiguousarray(a, dtype=np.float64)
    at = av if pretransposed else np.ascontiguousarray(av.T)
    bm = np.ascontiguousarray(bmat, dtype=np.float64)
    m, n1 = at.shape
    n2 = bm.shape[1]
    assert bm.shape[0] == m
    if words is None:
        words = draw_words(seed, d, b)
    h1, s1, h2, s2 = tables(words, d, b, n1, n2)
    starts, ends = chunk_bounds(m, threads)
    out = np.empty((d, b), dtype=np.float64)
    if transform == "fwht":
        rc = lib.oracle_compress_fwht(_p(at), _p(bm), m, n1, n2, _p(h1), _p(s1), _p(h2), _p(s2),
                                      d, b, _p(starts), _p(ends), threads, threads, _p(out))
    else:
        tw, twi, rev = fft_tables(b)
        tw = np.ascontiguousarray(tw)
        twi = np.ascontiguousarray(twi)
        rc = lib.oracle_compress_fft(_p(at), _p(bm), m, n1, n2, _p(h1), _p(s1), _p(h2), _p(s2),
                                     d, b, _p(tw), _p(twi), _p(rev), _p(starts), _p(ends),
                                     threads, threads, _p(out))
    if rc != 0:
        raise MemoryError("oracle compress allocation failed")
    return out


def accumulate_fwht(at: np.ndarray, bm: np.ndarray, *, b: int, d: int, words: np.ndarray,
                    k0: int, k1: int, threads: int = 1) -> np.ndarray:
    """Pre-inverse FWHT accumulator over inner indices [k0, k1) (the additive
    unit of the kernel, sketch.py:162-177) — used for bounded CPU-baseline
    samples and k-slice parity checks at full size."""
    lib = _load()
    at = np.ascontiguousarray(at, dtype=np.float64)
    bm = np.ascontiguousarray(bm, dtype=np.float64)
    n1 = at.shape[1]
    n2 = bm.shape[1]
    h1, s1, h2, s2 = tables(words, d, b, n1, n2)
    acc = np.zeros((d, b), dtype=np.float64)
    rc = lib.oracle_accumulate_fwht(_p(at), _p(bm), n1, n2, _p(h1), _p(s1), _p(h2), _p(s2),
                                    d, b, k0, k1, threads, _p(acc))
    if rc != 0:
        raise MemoryError("oracle accumulate allocation failed")
    return acc


def fwht_inverse_scaled(acc: np.ndarray) -> np.ndarray:
    """sketch.py:183-188: FWHT each row then * (1/b)."""
    lib = _load()
    out = np.ascontiguousarray(acc, dtype=np.float64).copy()
    d, b = out.shape
    for t in range(d):
        row = out[t]
        lib.oracle_fwht_inplace(_p(row), b)
    out *= 1.0 / b
    return out


def fwht(x: np.ndarray) -> np.ndarray:
    lib = _load()
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    lib.oracle_fwht_inplace(_p(y), y.shape[0])
    return y


def fft_forward_half(x: np.ndarray) -> np.ndarray:
    """transforms.py:130-138."""
    lib = _load()
    xv = np.ascontiguousarray(x, dtype=np.float64)
    n = xv.shape[0]
    tw, _, rev = fft_tables(n)
    z = xv.astype(np.complex128)
    lib.oracle_fft_inplace(_p(z), n, _p(np.ascontiguousarray(tw)), _p(rev))
    return z[: n // 2 + 1].copy()


def fft_inverse_half(spec: np.ndarray) -> np.ndarray:
    """transforms.py:141-165 (without the imag-part validation)."""
    lib = _load()
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    m = spec.shape[0]
    n = 2 * (m - 1)
    _, twi, rev = fft_tables(n)
    z = np.empty(n, dtype=np.complex128)
    z[:m] = spec
    z[m:] = np.conj(spec[-2:0:-1])
    lib.oracle_fft_inplace(_p(z), n, _p(np.ascontiguousarray(twi)), _p(rev))
    return z.real / n


def compress_slow(a, bmat, *, b: int, d: int, transform: str, seed: int) -> np.ndarray:
    """Reference tests/helpers.py:49-71: per-outer-product one-shot convolutions
    (np.add.at scatter).  Pure numpy; tiny sizes only."""
    a = np.asarray(a, dtype=np.float64)
    bmat = np.asarray(bmat, dtype=np.float64)
    words = draw_words(seed, d, b)
    h1, s1, h2, s2 = tables(words, d, b, a.shape[0], bmat.shape[1])
    m = a.shape[1]
    polys = np.zeros((d, b))
    for t in range(d):
        for k in range(m):
            pa = np.zeros(b)
            pb = np.zeros(b)
            np.add.at(pa, h1[t], s1[t] * a[:, k])
            np.add.at(pb, h2[t], s2[t] * bmat[k, :])
            if transform == "fwht":
                x, y = fwht(pa), fwht(pb)
                polys[t] += fwht(x * y) / b
            else:
                polys[t] += fft_inverse_half(fft_forward_half(pa) * fft_forward_half(pb))
    return polys


# --------------------------------------------------------------------------- decompress
def decompress(polys: np.ndarray, words: np.ndarray, *, b: int, d: int, transform: str,
               n1: int, n2: int, r0: int = 0, r1: int | None = None, want_est: bool = True,
               thr: float = 0.5, strict: bool = True, want_hh: bool = False, threads: int = 0):
    """Rows [r0, r1) of the estimate grid (sketch.py:375-399) plus the
    heavy-hitter count/list for |est| > thr (strict) or >= thr."""
    lib = _load()
    r1 = n1 if r1 is None else r1
    polys = np.ascontiguousarray(polys, dtype=np.float64)
    h1, s1, h2, s2 = tables(words, d, b, n1, n2)
    est = np.empty((r1 - r0, n2), dtype=np.float64) if want_est else None
    cnt = np.zeros(1, dtype=np.int64)
    lib.oracle_decompress(_p(polys), d, b, 1 if transform == "fwht" else 0, _p(h1), _p(s1), _p(h2),
                          _p(s2), n1, n2, r0, r1, _p(est) if est is not None else None,
                          float(thr), 1 if strict else 0, None, 0, _p(cnt), threads)
    hh = None
    if want_hh:
        hh = np.empty((int(cnt[0]), 2), dtype=np.int64)
        cnt2 = np.zeros(1, dtype=np.int64)
        lib.oracle_decompress(_p(polys), d, b, 1 if transform == "fwht" else 0, _p(h1), _p(s1),
                              _p(h2), _p(s2), n1, n2, r0, r1, None, float(thr), 1 if strict else 0,
                              _p(hh), int(cnt[0]), _p(cnt2), threads)
    return est, int(cnt[0]), hh


def cpu_count() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
