"""Seeded synthetic instances for the five BASELINE.json configurations.

BASELINE.json describes the constructions but not their seeds; the seeds are
fixed here and recorded in DESIGN.md.  The constructions are this repo's own
(the reference's ``instances.py`` generators do not produce them).  Every
random draw happens on the host with numpy (O(n) or O(nnz) values, except the
i.i.d. +-1 operands of cfg3 which are drawn as n*n bits), and the dense
operands are then assembled with elementwise float64 arithmetic in a fixed
order, so a host (numpy) build and a device (torch) build of the same config
are bit-identical.

Configs (BASELINE.json ``configs``):
  cfg1  n=1024  fwht b=2^12 d=3  A = H diag(s)/sqrt(n), B = A^T S, S: 64 nnz +-U[1,10]
  cfg2  n=4096  fft  b=2^14 d=5  same, S = signed permutation * U[1,10] (nnz = n)
  cfg3  n=16384 fwht b=2^16 d=5  A, B i.i.d. +-1; 256 planted columns B[:, j] = A[i, :]
  cfg4  n=32768 fwht b=2^18 d=7  Hadamard construction, S: 4096 nnz
  cfg5  n=8192  sweep b in 2^12..2^20, d in {3,5,9}, nnz in {512, 8192, 131072}, both variants
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INSTANCE_SEEDS = {"cfg1": 101, "cfg2": 102, "cfg3": 103, "cfg4": 104, "cfg5": 105}
SKETCH_SEEDS = {"cfg1": 201, "cfg2": 202, "cfg3": 203, "cfg4": 204, "cfg5": 205}


@dataclass
class Workload:
    name: str
    n: int
    b: int
    d: int
    transform: str
    sketch_seed: int
    threshold: float
    strict: bool
    big: np.ndarray  # (k, 2) int64 positions of the planted / nonzero product entries
    a: object = field(repr=False, default=None)
    bmat: object = field(repr=False, default=None)

    @property
    def log2b(self) -> int:
        return self.b.bit_length() - 1


CONFIGS = {
    "cfg1": dict(n=1024, b=1 << 12, d=3, transform="fwht", kind="hadamard", nnz=64, threshold=0.5),
    "cfg2": dict(n=4096, b=1 << 14, d=5, transform="fft", kind="hadamard_perm", nnz=4096, threshold=0.5),
    "cfg3": dict(n=16384, b=1 << 16, d=5, transform="fwht", kind="pm1_planted", nnz=256, threshold=8192.0),
    "cfg4": dict(n=32768, b=1 << 18, d=7, transform="fwht", kind="hadamard", nnz=4096, threshold=0.5),
}

CFG5_B = [1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20]
CFG5_D = [3, 5, 9]
CFG5_NNZ = [512, 8192, 131072]


def cfg5_name(b: int, d: int, nnz: int, transform: str) -> str:
    return f"cfg5_b{b.bit_length() - 1}_d{d}_nnz{nnz}_{transform}"


def _hadamard_signs(n: int, rng) -> np.ndarray:
    return 1.0 - 2.0 * rng.integers(0, 2, size=n).astype(np.float64)


def hadamard_matrix(n: int, xp=np, device=None):
    """Sylvester H[i, j] = (-1)^popcount(i & j) as float64."""
    if xp is np:
        h = np.ones((1, 1), dtype=np.int8)
        while h.shape[0] < n:
            h = np.block([[h, h], [h, -h]])
        return h.astype(np.float64)
    import torch
    i = torch.arange(n, device=device, dtype=torch.int64)
    x = i[:, None] & i[None, :]
    par = torch.zeros_like(x)
    while True:
        par ^= x & 1
        x = x >> 1
        if not bool(x.any()):
            break
    return (1 - 2 * par).to(torch.float64)


def _sparse_entries(n: int, nnz: int, rng, permutation: bool):
    if permutation:
        rows = np.arange(n, dtype=np.int64)
        cols = rng.permutation(n).astype(np.int64)
    else:
        flat = rng.choice(n * n, size=nnz, replace=False).astype(np.int64)
        rows, cols = flat // n, flat % n
    mags = rng.uniform(1.0, 10.0, size=rows.shape[0])
    sgn = 1.0 - 2.0 * rng.integers(0, 2, size=rows.shape[0]).astype(np.float64)
    vals = sgn * mags
    order = np.lexsort((rows, cols))  # by column, then row
    return rows[order], cols[order], vals[order]


def _rounds(cols: np.ndarray):
    """Split entries (sorted by column) into rounds with distinct columns, so
    B[:, cols] += ... never aliases inside a round (fixed accumulation order)."""
    rank = np.zeros(cols.shape[0], dtype=np.int64)
    for q in range(1, cols.shape[0]):
        rank[q] = rank[q - 1] + 1 if cols[q] == cols[q - 1] else 0
    return [np.nonzero(rank == r)[0] for r in range(int(rank.max()) + 1 if cols.size else 0)]


def _hadamard_instance(n: int, nnz: int, seed: int, permutation: bool, xp=np, device=None):
    rng = np.random.default_rng(seed)
    s = _hadamard_signs(n, rng)
    rows, cols, vals = _sparse_entries(n, nnz, rng, permutation)
    inv = 1.0 / np.sqrt(float(n))
    if xp is np:
        a = hadamard_matrix(n) * s[None, :]
        a *= inv
        bm = np.zeros((n, n), dtype=np.float64)
        for idx in _rounds(cols):
            bm[:, cols[idx]] += (a[rows[idx], :] * vals[idx][:, None]).T
    else:
        import torch
        a = hadamard_matrix(n, torch, device) * torch.as_tensor(s, device=device)[None, :]
        a *= inv
        bm = torch.zeros((n, n), dtype=torch.float64, device=device)
        for idx in _rounds(cols):
            r = torch.as_tensor(rows[idx], device=device)
            c = torch.as_tensor(cols[idx], device=device)
            v = torch.as_tensor(vals[idx], device=device)
            bm[:, c] += (a[r, :] * v[:, None]).T
    big = np.stack([rows, cols], axis=1)
    return a, bm, big


def _pm1_planted(n: int, nplant: int, seed: int, xp=np, device=None):
    rng = np.random.default_rng(seed)
    abits = rng.integers(0, 2, size=(n, n), dtype=np.uint8)
    bbits = rng.integers(0, 2, size=(n, n), dtype=np.uint8)
    pi = rng.choice(n, size=nplant, replace=False).astype(np.int64)
    pj = rng.choice(n, size=nplant, replace=False).astype(np.int64)
    if xp is np:
        a = 1.0 - 2.0 * abits.astype(np.float64)
        bm = 1.0 - 2.0 * bbits.astype(np.float64)
        bm[:, pj] = a[pi, :].T
    else:
        import torch
        a = 1.0 - 2.0 * torch.as_tensor(abits, device=device).to(torch.float64)
        bm = 1.0 - 2.0 * torch.as_tensor(bbits, device=device).to(torch.float64)
        bm[:, torch.as_tensor(pj, device=device)] = a[torch.as_tensor(pi, device=device), :].T
    big = np.stack([pi, pj], axis=1)
    return a, bm, big


def make(name: str, xp=np, device=None, with_data: bool = True) -> Workload:
    """Build config ``name`` ("cfg1".."cfg4" or a cfg5_* point name)."""
    if name.startswith("cfg5_"):
        parts = name.split("_")
        b = 1 << int(parts[1][1:])
        d = int(parts[2][1:])
        nnz = int(parts[3][3:])
        transform = parts[4]
        n = 8192
        w = Workload(name, n, b, d, transform, SKETCH_SEEDS["cfg5"], 0.5, True, np.zeros((0, 2), np.int64))
        if with_data:
            # the operands depend on nnz only (seeded per nnz), not on (b, d, transform)
            w.a, w.bmat, w.big = _hadamard_instance(n, nnz, INSTANCE_SEEDS["cfg5"] * 1000 + nnz, False, xp, device)
        return w
    c = CONFIGS[name]
    w = Workload(name, c["n"], c["b"], c["d"], c["transform"], SKETCH_SEEDS[name], c["threshold"], True,
                 np.zeros((0, 2), np.int64))
    if not with_data:
        return w
    if c["kind"] == "hadamard":
        w.a, w.bmat, w.big = _hadamard_instance(c["n"], c["nnz"], INSTANCE_SEEDS[name], False, xp, device)
    elif c["kind"] == "hadamard_perm":
        w.a, w.bmat, w.big = _hadamard_instance(c["n"], c["nnz"], INSTANCE_SEEDS[name], True, xp, device)
    else:
        w.a, w.bmat, w.big = _pm1_planted(c["n"], c["nnz"], INSTANCE_SEEDS[name], xp, device)
    return w


def all_cfg5_points():
    for transform in ("fwht", "fft"):
        for b in CFG5_B:
            for d in CFG5_D:
                for nnz in CFG5_NNZ:
                    yield cfg5_name(b, d, nnz, transform)
