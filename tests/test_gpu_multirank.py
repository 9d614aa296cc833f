"""Multi-rank path on the GPU: the k-sharded compress through the real kernels
and a real torch.distributed collective.

The pool exposes one GPU per call, and NCCL refuses two ranks on one device, so
two views are tested here:
  * NCCL, world size 1: the one allreduce of compress_sharded goes through an
    NCCL communicator on cuda:0 (the plumbing the N-GPU bench uses);
  * gloo, world size 2 on cuda:0: each rank compresses its own k-slab with the
    CUDA kernels, the accumulators meet in one gloo allreduce (host-staged, so
    no kernel waits on another rank's kernel), every rank extracts its own row
    block and rank 0 gathers the heavy-hitter list.  Integer data: the sharded
    sketch must equal the single-process one bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2601_09477_b200 as P
from paper_2601_09477_b200 import _device
from paper_2601_09477_b200 import distributed as D

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance(n, seed=3):
    rng = np.random.default_rng(seed)
    a = rng.integers(-4, 5, size=(n, n)).astype(np.float64)
    bm = rng.integers(-4, 5, size=(n, n)).astype(np.float64)
    # two planted heavy entries well above the background
    a[5, :] = 1.0
    bm[:, 9] = 1.0
    return a, bm


def test_nccl_world1_compress_sharded_matches_compress():
    port = _free_port()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a, bm = _instance(1024)
        p = P.SketchParams(n=1024, b=1 << 14, d=5, seed=11)
        ref = P.compress(a, bm, p)
        ad = torch.as_tensor(a, device="cuda")
        bd = torch.as_tensor(bm, device="cuda")
        calls = []

        def nccl_sum(t):
            calls.append(t.numel())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        sk = D.compress_sharded(ad, bd, p, n_rows=1024, n_cols=1024, a_layout=_device.KMINOR, all_reduce=nccl_sum)
        assert calls == [p.d * p.b]
        assert np.array_equal(sk.polys, ref.polys)
        est, pairs = P.extract_all(sk, 600.0, strict=True)
        hh = D.gather_heavy_hitters(pairs)
        assert np.array_equal(hh.cpu().numpy(), P.heavy_hitters(ref, 600.0, strict=True))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, transform, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n = 2048
        a, bm = _instance(n)
        p = P.SketchParams(n=n, b=1 << 14, d=3, transform=transform, seed=17)
        k0, k1 = D.shard_bounds(n, world, rank)
        r0, r1 = D.row_bounds(n, world, rank)
        a_slab = torch.as_tensor(a, device="cuda")[:, k0:k1]  # column view: k-minor, no copy
        b_slab = torch.as_tensor(bm[k0:k1], device="cuda")

        def host_sum(t):  # gloo reduces host tensors; the accumulator goes down and back once
            c = t.cpu()
            dist.all_reduce(c, op=dist.ReduceOp.SUM)
            t.copy_(c)

        sk = D.compress_sharded(a_slab, b_slab, p, n_rows=n, n_cols=n, a_layout=_device.KMINOR, all_reduce=host_sum)
        thr = 900.0
        est, pairs = P.extract_all(sk, thr, strict=True, r0=r0, r1=r1)
        got = D.gather_heavy_hitters(pairs.cpu())
        q.put((rank, sk.polys, est.cpu().numpy(), None if got is None else got.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transform", ["fwht", "fft"])
def test_gloo_world2_sharded_path_on_one_gpu(transform):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, transform, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    n = 2048
    a, bm = _instance(n)
    p = P.SketchParams(n=n, b=1 << 14, d=3, transform=transform, seed=17)
    ref = P.compress(a, bm, p)
    cn = float(np.linalg.norm(a @ bm))
    for rank, polys, est, _ in res:
        if transform == "fwht":
            assert np.array_equal(polys, ref.polys), rank  # integer data: exact in any order
        else:
            assert np.max(np.abs(polys - ref.polys)) <= 1e-10 * cn, rank
    est_ref, hh_ref = P.extract_all(ref, 900.0, strict=True)
    est_ref = est_ref.cpu().numpy()
    r0, r1 = D.row_bounds(n, world, 0)
    assert np.max(np.abs(res[0][2] - est_ref[r0:r1])) <= 1e-10 * cn
    r0, r1 = D.row_bounds(n, world, 1)
    assert np.max(np.abs(res[1][2] - est_ref[r0:r1])) <= 1e-10 * cn
    assert res[1][3] is None
    if transform == "fwht":
        assert np.array_equal(res[0][3], hh_ref.cpu().numpy())
        assert res[0][3].shape[0] >= 1
