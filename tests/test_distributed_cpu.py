"""Multi-rank host logic on CPU with gloo, world_size 2 (CPU-only).

The GPU path shards the inner dimension k across ranks, each rank producing
the pre-inverse accumulator of its slab, and joins them with ONE sum
allreduce (paper_2601_09477_b200.distributed.reduce_accumulator).  Here the
per-rank accumulators come from the CPU oracle (the checker), the collective is
the real torch.distributed all_reduce over gloo, and the result must equal the
single-process reference sketch bit for bit (integer data: every partial sum
is exact, so summation order cannot matter).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sketch_oracle as O
from paper_2601_09477_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        n, b, d = 40, 64, 3
        a = rng.integers(-3, 4, size=(n, n)).astype(np.float64)
        bm = rng.integers(-3, 4, size=(n, n)).astype(np.float64)
        words = O.draw_words(7, d, b)
        at = np.ascontiguousarray(a.T)
        k0, k1 = D.shard_bounds(n, world, rank)
        acc = O.accumulate_fwht(at[k0:k1], bm[k0:k1], b=b, d=d, words=words, k0=0, k1=k1 - k0)
        t = torch.from_numpy(acc)
        D.reduce_accumulator(t)
        polys = O.fwht_inverse_scaled(t.numpy())
        ref = O.compress(a, bm, b=b, d=d, transform="fwht", seed=7, threads=1)
        r0, r1 = D.row_bounds(n, world, rank)
        est, _, _ = O.decompress(polys, words, b=b, d=d, transform="fwht", n1=n, n2=n, r0=r0, r1=r1)
        est_ref, _, _ = O.decompress(ref, words, b=b, d=d, transform="fwht", n1=n, n2=n)
        # heavy hitters: each rank thresholds its own rows, rank 0 collects the global list
        thr = float(np.quantile(np.abs(est_ref), 0.9))
        ii, jj = np.nonzero(np.abs(est) > thr)
        local = torch.from_numpy(np.stack([ii + r0, jj], axis=1).astype(np.int64))
        got = D.gather_heavy_hitters(local)
        gi, gj = np.nonzero(np.abs(est_ref) > thr)
        want = np.stack([gi, gj], axis=1)
        hh_ok = (got is None) if rank else bool(np.array_equal(got.numpy(), want))
        q.put((rank, bool(np.array_equal(polys, ref)), bool(np.array_equal(est, est_ref[r0:r1])) and hh_ok))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for m in (0, 1, 7, 1000, 16384, 16400, 32768 + 5):
        for world in (1, 2, 3, 5, 8):
            parts = [D.shard_bounds(m, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            # every slab starts on a 32-index k-tile boundary; whole tiles split evenly
            assert all(p[0] % 32 == 0 for p in parts)
            tiles = [-(-(p[1] - p[0]) // 32) for p in parts]
            assert max(tiles) - min(tiles) <= 1
            rows = [D.row_bounds(m, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == m
            assert max(r[1] - r[0] for r in rows) - min(r[1] - r[0] for r in rows) <= 1
    plan = D.plan_shards(16384, 16384, 8)
    assert [p["k1"] - p["k0"] for p in plan] == [2048] * 8


def test_gloo_world2_allreduce_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r[0] for r in results) == [0, 1]
    assert all(r[1] and r[2] for r in results), results


def test_reduce_accumulator_single_process_is_identity():
    t = torch.arange(6, dtype=torch.float64)
    assert torch.equal(D.reduce_accumulator(t.clone()), t)
    calls = []
    D.reduce_accumulator(t, all_reduce=lambda x: calls.append(x.numel()))
    assert calls == [6]
