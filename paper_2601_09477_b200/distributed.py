"""Multi-GPU sketched product: inner-dimension (k) sharding, one allreduce.

P = sum_k (per-k sketch products) is a sum of independent units, so rank g of
G owns inner indices [k_lo(g), k_hi(g)) — the k-slab A[:, slab] (as rows of
A^T) and B[slab, :] — and produces the pre-inverse accumulator of its slab with
the same kernel as the single-GPU path.  The only exchange is one sum-allreduce
of that accumulator (d x b float64 for FWHT, d x (b/2+1) complex for FFT; the
reference's fixed-order chunk reduction sketch.py:178-182 / 219-223), over NCCL
on NVLink / NVSwitch.  Every rank then runs the cheap inverse redundantly and
extracts its own block of output rows (row-sharded step 5, no exchange).

Works with any torch.distributed backend whose all_reduce supports CUDA
tensors (nccl on GPUs); the CPU tests drive the same host logic with gloo.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidParameterError
from .sketch import ProductSketch, SketchParams, _drawn, effective_threads


K_TILE = 32  # inner indices per k-tile of the compress kernels


def _balanced(m: int, world: int, rank: int) -> tuple[int, int]:
    edges = np.linspace(0, m, world + 1).astype(np.int64)
    return int(edges[rank]), int(edges[rank + 1])


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous k-slab of rank ``rank``: whole 32-index k-tiles split as evenly as
    possible (slabs then start on tile boundaries and keep the 16-byte pair mapping
    of the compress kernels; the last rank also takes the partial tail tile)."""
    if world < 1 or not (0 <= rank < world):
        raise InvalidParameterError(f"bad rank {rank} for world size {world}")
    tiles = -(-m // K_TILE)
    t0, t1 = _balanced(tiles, world, rank)
    return min(m, t0 * K_TILE), min(m, t1 * K_TILE)


def row_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block of output rows (step 5 is row-sharded)."""
    if world < 1 or not (0 <= rank < world):
        raise InvalidParameterError(f"bad rank {rank} for world size {world}")
    return _balanced(n_rows, world, rank)


def compress_sharded(a_slab, b_slab, params: SketchParams, n_rows: int | None = None, n_cols: int | None = None,
                     group=None, threads: int | None = None, all_reduce=None, a_layout: int = 0) -> ProductSketch:
    """Sketch of A @ B from this rank's k-slab; returns the full sketch on every rank.

    a_slab: this rank's slab of A — rows of A^T (``a_layout=0``, k-major, shape
    (k_local, n1)) or a column view A[:, k0:k1] (``a_layout=1``, k-minor, shape
    (n1, k_local), used without a copy); b_slab: B[k0:k1] (k_local, n2).
    ``all_reduce`` (default: torch.distributed.all_reduce with SUM) is the one
    collective of the path.
    """
    from . import _device

    effective_threads(threads)
    kl = a_slab.shape[1] if a_layout == _device.KMINOR else a_slab.shape[0]
    n1 = a_slab.shape[0] if a_layout == _device.KMINOR else a_slab.shape[1]
    if kl != b_slab.shape[0]:
        raise InvalidParameterError(f"inner slabs must match, got {kl} and {b_slab.shape[0]}")
    hashes, words = _drawn(int(params.seed), params.d, params.b)
    if not getattr(a_slab, "is_cuda", False) and not getattr(b_slab, "is_cuda", False):
        # host slabs: streamed upload overlapped with the compress kernel
        acc = _device.compress_host(_device.host_f64(a_slab), _device.host_f64(b_slab), words,
                                    params.d, params.log2b, params.transform, a_layout, _device.require_cuda())
    else:
        acc = _device.compress_accumulate(a_slab, b_slab, words, params.d, params.log2b,
                                          params.transform, 0, kl, a_layout=a_layout)
    reduce_accumulator(acc, group=group, all_reduce=all_reduce)
    polys = _device.finalize(acc, params.d, params.log2b, params.transform)
    return ProductSketch(polys=polys, hashes=hashes, params=params,
                         n_rows=n_rows if n_rows is not None else n1,
                         n_cols=n_cols if n_cols is not None else b_slab.shape[1])


def reduce_accumulator(acc, group=None, all_reduce=None):
    """The path's single exchange: elementwise sum of the ranks' accumulators."""
    import torch.distributed as dist

    if all_reduce is not None:
        all_reduce(acc)
    elif dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def gather_heavy_hitters(pairs, dst: int = 0, group=None):
    """Collect the row-sharded heavy-hitter lists on rank ``dst``.

    Rank g extracted output rows [g n/G, (g+1) n/G), so its pairs are already in
    row-major order and concatenating the ranks' lists in rank order is the
    global row-major list.  One all_gather of the counts, one of the lists padded
    to the largest count (all_gather works on every backend, gather does not).
    Returns the (k, 2) int64 tensor on ``dst`` and None elsewhere.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return pairs
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pairs = pairs.to(torch.int64).reshape(-1, 2)
    cnt = torch.tensor([pairs.shape[0]], dtype=torch.int64, device=pairs.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    padded = torch.zeros((max(counts), 2), dtype=torch.int64, device=pairs.device)
    padded[:pairs.shape[0]] = pairs
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    if rank != dst:
        return None
    return torch.cat([buf[:c] for buf, c in zip(bufs, counts)])


def plan_shards(m: int, n_rows: int, world: int) -> list[dict]:
    """Host-side description of every rank's k-slab and output-row block."""
    out = []
    for r in range(world):
        k0, k1 = shard_bounds(m, world, r)
        r0, r1 = row_bounds(n_rows, world, r)
        out.append({"rank": r, "k0": k0, "k1": k1, "r0": r0, "r1": r1})
    return out
