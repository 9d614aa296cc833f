"""GPU parity: the CUDA path (through the C ABI) against the reference goldens
and the CPU oracle.  Run on a B200 with ``pytest -m gpu``.

Tolerances (BASELINE north star): hash buckets/signs bit-exact; sketch values
and estimates within 1e-10 * ||C||_F; heavy-hitter sets identical.  cfg3 is
integer-valued, so its sketch must be bit-identical to the reference.
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2601_09477_b200 as P
from conftest import cfg_golden
from oracle import sketch_oracle as O
from paper_2601_09477_b200 import _device
from paper_2601_09477_b200 import workloads as W
from paper_2601_09477_b200.hashing import SketchHashes

pytestmark = pytest.mark.gpu
TOL = 1e-10  # relative to ||C||_F


def _sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def _cnorm(a, bm):
    return float(np.linalg.norm(np.asarray(a) @ np.asarray(bm)))


def test_native_library_loaded_and_kernels_run():
    from paper_2601_09477_b200 import _lib

    lib = _lib.load()
    assert lib.smm_abi_version() == 1
    sk = P.compress(np.eye(4), np.eye(4), P.SketchParams(n=4, b=16, d=1, seed=5))
    assert isinstance(sk.polys_device(), torch.Tensor) and sk.polys_device().is_cuda


def test_small_cases_match_reference(small_cases):
    for c in small_cases:
        p = P.SketchParams(n=c["m"], b=c["b"], d=c["d"], transform=c["transform"], seed=c["seed"])
        rect = c["n1"] != c["m"] or c["n2"] != c["m"]
        sk = P.compress_rect(c["a"], c["bm"], p) if rect else P.compress(c["a"], c["bm"], p, threads=c["threads"])
        assert np.array_equal(sk.words, c["words"])
        scale = max(1.0, _cnorm(c["a"], c["bm"]))
        assert np.max(np.abs(sk.polys - c["polys"])) <= TOL * scale, c["name"]
        est = P.decompress_all(sk)
        assert est.shape == c["est"].shape
        assert np.max(np.abs(est - c["est"])) <= TOL * scale, c["name"]


def test_hash_tables_bit_exact(hash_golden):
    for tab in hash_golden["tables"]:
        a, c, shift = int(tab["a"]), int(tab["c"]), tab["shift"]
        b = 1 << (64 - shift)
        words = np.array([a, c, a, c, a, c, a, c], dtype=np.uint64)
        h = SketchHashes.from_words(words, 1, b)
        buckets = _device.hash_table(h, 0, 2000).cpu().numpy().astype(np.int64)[0]
        signs = _device.hash_table(h, 2, 2000).cpu().numpy().astype(int)[0]
        assert buckets.tolist() == tab["buckets"]
        assert signs.tolist() == tab["signs"]


def test_hash_tables_match_oracle_on_config_sizes():
    for seed, d, b, n in ((203, 5, 1 << 16, 16384), (204, 7, 1 << 18, 32768), (7, 3, 1 << 32, 5000)):
        words = O.draw_words(seed, d, b)
        h = SketchHashes.from_words(words, d, b)
        h1, s1, h2, s2 = O.tables(words, d, b, n, n)
        assert np.array_equal(_device.hash_table(h, 0, n).cpu().numpy().astype(np.int64), h1)
        assert np.array_equal(_device.hash_table(h, 1, n).cpu().numpy().astype(np.int64), h2)
        assert np.array_equal(_device.hash_table(h, 2, n).cpu().numpy().astype(np.float64), s1)
        assert np.array_equal(_device.hash_table(h, 3, n).cpu().numpy().astype(np.float64), s2)


# every BASELINE point (cfg1-3 and all 90 points of the cfg5 sweep) against its reference
# golden (tools/make_golden.py); a missing golden is a failure, not a skip
CONFIGS = ["cfg1", "cfg2", "cfg3"] + [W.cfg5_name(b, d, nnz, tr) for b in W.CFG5_B for d in W.CFG5_D
                                      for nnz in W.CFG5_NNZ for tr in ("fwht", "fft")]


@pytest.mark.parametrize("name", CONFIGS)
def test_config_matches_reference(name):
    g = cfg_golden(name)
    assert g is not None, f"no reference golden for BASELINE point {name} (tools/make_golden.py)"
    w = W.make(name, xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    sk = P.compress(w.a, w.bmat, p)
    assert np.array_equal(sk.words, g["words"])
    cn = float(g["cnorm"][0])
    if not np.isfinite(cn):
        cn = float(torch.linalg.norm(w.a @ w.bmat))
    polys = sk.polys
    if name == "cfg3":
        assert _sha(polys) == bytes(g["polys_sha256"]).decode()  # integer-exact: bit-identical
    elif "polys" in g:
        assert np.max(np.abs(polys - g["polys"])) <= TOL * cn
    samp = np.take_along_axis(polys, g["polys_sample_idx"], axis=1)
    assert np.max(np.abs(samp - g["polys_sample"])) <= TOL * cn
    assert np.allclose(polys.sum(axis=1), g["polys_rowsum"], rtol=0, atol=TOL * cn * w.b)
    est = P.decompress_rows(sk)
    ij = torch.as_tensor(g["est_sample_ij"], device="cuda")
    e = est[ij[:, 0], ij[:, 1]].cpu().numpy()
    assert np.max(np.abs(e - g["est_sample"])) <= TOL * cn
    # row sums of the full estimate grid (each estimate within TOL * cn, n2 per row)
    assert np.max(np.abs(est.sum(dim=1).cpu().numpy() - g["est_rowsum"])) <= TOL * cn * w.n
    big = torch.as_tensor(w.big, device="cuda")
    if big.numel():
        eb = est[big[:, 0], big[:, 1]].cpu().numpy()
        assert np.max(np.abs(eb - g["est_big"])) <= TOL * cn
    del est
    hh = P.heavy_hitters(sk, w.threshold, strict=True)
    assert hh.shape[0] == int(g["hh_count"][0])
    assert _sha(hh.astype(np.int64)) == bytes(g["hh_sha256"]).decode()


def test_cfg3_k_slices_add_exactly():
    # the multi-GPU unit: accumulators of disjoint k-slabs sum to the full one (exact: integer data)
    w = W.make("cfg3", xp=torch, device="cuda")
    words = O.draw_words(w.sketch_seed, w.d, w.b)
    at = _device.transpose(w.a)
    full = _device.compress_accumulate(at, w.bmat, words, w.d, w.log2b, "fwht", 0, w.n)
    world = 8
    parts = torch.zeros_like(full)
    for r in range(world):
        k0, k1 = r * w.n // world, (r + 1) * w.n // world
        parts += _device.compress_accumulate(at[k0:k1], w.bmat[k0:k1], words, w.d, w.log2b, "fwht", 0, k1 - k0)
    assert torch.equal(parts, full)
    # and a slab against the CPU oracle (bounded size)
    k0, k1 = 1000, 1016
    acc = _device.compress_accumulate(at, w.bmat, words, w.d, w.log2b, "fwht", k0, k1).cpu().numpy()
    ref = O.accumulate_fwht(at[k0:k1].cpu().numpy(), w.bmat[k0:k1].cpu().numpy(), b=w.b, d=w.d, words=words,
                            k0=0, k1=k1 - k0, threads=8)
    assert np.array_equal(acc, ref)


def test_cfg4_full_size_properties():
    w = W.make("cfg4", xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    words = O.draw_words(p.seed, p.d, p.b)
    at = _device.transpose(w.a)
    cn = float(torch.linalg.norm(w.a @ w.bmat))  # ||C||_F (C = S up to rounding)
    # k-slab vs the CPU oracle
    k0, k1 = 4096, 4104
    acc = _device.compress_accumulate(at, w.bmat, words, p.d, p.log2b, "fwht", k0, k1).cpu().numpy()
    ref = O.accumulate_fwht(at[k0:k1].cpu().numpy(), w.bmat[k0:k1].cpu().numpy(), b=w.b, d=w.d, words=words,
                            k0=0, k1=k1 - k0, threads=8)
    assert np.max(np.abs(acc - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())
    # 8-way k-sharded accumulate == single-GPU accumulate (only the summation order differs)
    full = _device.compress_accumulate(at, w.bmat, words, p.d, p.log2b, "fwht", 0, w.n)
    parts = torch.zeros_like(full)
    for r in range(8):
        a0, a1 = r * w.n // 8, (r + 1) * w.n // 8
        parts += _device.compress_accumulate(at[a0:a1], w.bmat[a0:a1], words, p.d, p.log2b, "fwht", 0, a1 - a0)
    polys = _device.finalize(full, p.d, p.log2b, "fwht")
    polys8 = _device.finalize(parts, p.d, p.log2b, "fwht")
    assert float((polys - polys8).abs().max()) <= TOL * cn
    sk = P.ProductSketch(polys, SketchHashes.from_words(words, p.d, p.b), p, w.n, w.n)
    est = P.decompress_rows(sk)
    big = torch.as_tensor(w.big, device="cuda")
    assert float((est[big[:, 0], big[:, 1]].abs() > 0.5).float().mean()) > 0.95
    g = cfg_golden("cfg4")
    assert g is not None, "no reference golden for cfg4"
    samp = np.take_along_axis(sk.polys, g["polys_sample_idx"], axis=1)
    assert np.max(np.abs(samp - g["polys_sample"])) <= TOL * cn
    assert np.allclose(sk.polys.sum(axis=1), g["polys_rowsum"], rtol=0, atol=TOL * cn * w.b)
    # estimates: the golden's 4096 sampled entries and every row sum of the n x n grid
    ij = torch.as_tensor(g["est_sample_ij"], device="cuda")
    assert np.max(np.abs(est[ij[:, 0], ij[:, 1]].cpu().numpy() - g["est_sample"])) <= TOL * cn
    assert np.max(np.abs(est.sum(dim=1).cpu().numpy() - g["est_rowsum"])) <= TOL * cn * w.n
    assert np.max(np.abs(est[big[:, 0], big[:, 1]].cpu().numpy() - g["est_big"])) <= TOL * cn
    del est
    hh = P.heavy_hitters(sk, w.threshold, strict=True)
    assert hh.shape[0] == int(g["hh_count"][0])
    assert _sha(hh.astype(np.int64)) == bytes(g["hh_sha256"]).decode()


def test_determinism_and_threads_independence():
    rng = np.random.default_rng(14)
    a, m = rng.normal(size=(96, 96)), rng.normal(size=(96, 96))
    for tr in ("fwht", "fft"):
        p = P.SketchParams(n=96, b=1 << 14, d=3, transform=tr, seed=15)
        s1 = P.compress(a, m, p, threads=1).polys
        s2 = P.compress(a, m, p, threads=5).polys
        assert np.array_equal(s1, s2)


def test_pretransposed_agrees_bitwise():
    rng = np.random.default_rng(5)
    a, m = rng.normal(size=(300, 300)), rng.normal(size=(300, 300))
    for tr, b in (("fwht", 1 << 13), ("fwht", 1 << 16), ("fft", 1 << 12)):
        p = P.SketchParams(n=300, b=b, d=3, transform=tr, seed=8)
        assert np.array_equal(P.compress(a, m, p).polys, P.compress_pretransposed(np.ascontiguousarray(a.T), m, p).polys)


def test_large_width_and_depth_against_oracle():
    # b up to 2^20 (cfg5 range) and d = 37 (reference acceptance criterion 5 depth)
    rng = np.random.default_rng(21)
    for n, b, d, tr in ((256, 1 << 20, 3, "fwht"), (128, 1 << 18, 5, "fft"), (200, 512, 37, "fwht"),
                        (200, 512, 37, "fft"), (1000, 1 << 13, 9, "fwht"), (700, 1 << 15, 1, "fwht")):
        a, m = rng.normal(size=(n, n)), rng.normal(size=(n, n))
        p = P.SketchParams(n=n, b=b, d=d, transform=tr, seed=31)
        got = P.compress(a, m, p).polys
        ref = O.compress(a, m, b=b, d=d, transform=tr, seed=31, threads=8)
        cn = _cnorm(a, m)
        assert np.max(np.abs(got - ref)) <= TOL * cn, (n, b, d, tr)
        est = P.decompress_all(P.compress(a, m, p))
        eref, _, _ = O.decompress(ref, O.draw_words(31, d, b), b=b, d=d, transform=tr, n1=n, n2=n)
        assert np.max(np.abs(est - eref)) <= TOL * cn


def test_heavy_hitter_comparators_and_order():
    # polys engineered so estimates hit the threshold exactly: strict excludes, inclusive includes
    b, d = 16, 3
    words = np.array([1 << 60, 0] * 3 + [1 << 60, 0] * 3 + [0, 0] * 6, dtype=np.uint64)  # bucket(x)=x, sign +1
    hashes = SketchHashes.from_words(words, d, b)
    polys = np.tile(np.array([0.5, -0.5, 0.25, 1.0, -2.0, 0.5, 0.0, 3.0] * 2), (d, 1))
    p = P.SketchParams(n=4, b=b, d=d, seed=0)
    sk = P.ProductSketch(polys, hashes, p, 4, 4)
    est = P.decompress_all(sk)
    for strict in (True, False):
        got = P.heavy_hitters(sk, 0.5, strict=strict)
        _, cnt, ref = O.decompress(polys, words, b=b, d=d, transform="fwht", n1=4, n2=4, thr=0.5, strict=strict,
                                   want_hh=True)
        assert np.array_equal(got, ref) and got.shape[0] == cnt
        mask = np.abs(est) > 0.5 if strict else np.abs(est) >= 0.5
        assert np.array_equal(got, np.argwhere(mask))
    assert P.heavy_hitters(sk, 0.5, strict=False).shape[0] > P.heavy_hitters(sk, 0.5, strict=True).shape[0]


def test_row_sharded_extraction_matches_full():
    rng = np.random.default_rng(3)
    a, m = rng.normal(size=(257, 257)), rng.normal(size=(257, 257))
    sk = P.compress(a, m, P.SketchParams(n=257, b=1 << 12, d=5, seed=2))
    full = P.decompress_rows(sk)
    for r0, r1 in ((0, 100), (100, 257), (37, 38), (5, 5)):
        part = P.decompress_rows(sk, r0, r1)
        assert torch.equal(part, full[r0:r1])
        hh = P.heavy_hitters(sk, 1.0, r0=r0, r1=r1)
        ref = np.argwhere(np.abs(full[r0:r1].cpu().numpy()) > 1.0)
        ref[:, 0] += r0
        assert np.array_equal(hh, ref)


def test_empty_k_range_gives_zero_accumulator():
    words = O.draw_words(1, 3, 1 << 13)
    at = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    for tr in ("fwht", "fft"):
        acc = _device.compress_accumulate(at, at, words, 3, 13, tr, 4, 4)
        assert float(acc.abs().max()) == 0.0


def test_transforms_api(transforms_golden):
    g = transforms_golden
    assert P.fwht_inplace(np.array([1.0, 2, 3, 4])).tolist() == [10, -2, -4, 0]
    assert np.allclose(P.xor_convolve([1, 2], [3, 4]), [11, 10])
    assert np.allclose(P.cyclic_convolve([1, 2], [3, 4]), [11, 10])
    assert np.allclose(P.fft_forward([0, 1, 0, 0]), [1, -1j, -1], atol=1e-12)
    for bstr, v in g["vectors"].items():
        x, y = np.array(v["x"]), np.array(v["y"])
        assert np.array_equal(P.fwht_inplace(x.copy()), np.array(v["fwht"]))
        assert np.allclose(P.xor_convolve(x, y), v["xor"], rtol=0, atol=1e-12 * max(1, np.abs(v["xor"]).max()))
        assert np.allclose(P.cyclic_convolve(x, y), v["cyc"], rtol=0, atol=1e-11 * max(1, np.abs(v["cyc"]).max()))
        z = P.fft_forward(x)
        assert np.allclose(z.real, v["fft_re"], atol=1e-11) and np.allclose(z.imag, v["fft_im"], atol=1e-11)
    with pytest.raises(P.InvalidSpectrumError):
        P.fft_inverse([1 + 1e-3j, 0, 1])
    with pytest.raises(P.InvalidParameterError):
        P.fwht_inplace(np.zeros(6))


@pytest.mark.parametrize("transform,log2b", [("fwht", 12), ("fwht", 6), ("fft", 10), ("fft", 15)])
def test_host_streamed_compress(transform, log2b):
    # host operands are uploaded in k-slabs while earlier slabs compute; every slab
    # after the first runs in accumulate mode.  The two-pass FWHT kernel continues
    # the single call's k order exactly; the other kernels add a slab accumulator.
    rng = np.random.default_rng(7)
    n1, m, n2 = 700, 1000, 650
    a = rng.standard_normal((n1, m))
    b = rng.standard_normal((m, n2))
    words = O.draw_words(11, 5, 1 << log2b)
    dev = torch.device("cuda")
    ref = _device.compress_accumulate(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), words, 5, log2b,
                                      transform, 0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    a_h = torch.from_numpy(a).pin_memory()
    b_h = torch.from_numpy(b).pin_memory()
    for chunk in (64, 96, 1024):
        got = _device.compress_host(a_h, b_h, words, 5, log2b, transform, _device.KMINOR, dev, chunk=chunk)
        if transform == "fwht" and log2b >= 8:
            assert torch.equal(got, ref)
        else:
            scale = float(ref.abs().max())
            assert float((got - ref).abs().max()) <= 1e-12 * scale
    # A^T given (k-major): the k-slab is a row block of the host array
    at_h = torch.from_numpy(np.ascontiguousarray(a.T))
    got = _device.compress_host(at_h, b_h, words, 5, log2b, transform, _device.KMAJOR, dev, chunk=128)
    scale = float(ref.abs().max())
    assert float((got - ref).abs().max()) <= 1e-12 * scale


def test_public_api_host_operands_bitwise_equal_to_device_operands():
    w = W.make("cfg1", xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    dev_sk = P.compress(w.a, w.bmat, p)
    host_sk = P.compress(w.a.cpu().pin_memory(), w.bmat.cpu(), p)
    np_sk = P.compress(w.a.cpu().numpy(), w.bmat.cpu().numpy(), p)
    assert np.array_equal(dev_sk.polys, host_sk.polys)
    assert np.array_equal(dev_sk.polys, np_sk.polys)


@pytest.mark.parametrize("d", [3, 9])
def test_one_pass_fft_host_streamed_bitwise_and_oracle(d):
    """fft1p (b = 2^12, rectangular, non-integer data): host operands streamed in k-slabs
    (SMM_FLAG_ACCUMULATE) give the device call's bits; polys and estimates against the CPU
    oracle within the north star's 1e-10 * ||C||_F; d = 9 runs as two launches."""
    from oracle import sketch_oracle as O
    from paper_2601_09477_b200 import _device

    rng = np.random.default_rng(17 + d)
    n1, m, n2 = 700, 1000, 900
    a = rng.standard_normal((n1, m))
    bm = rng.standard_normal((m, n2))
    p = P.SketchParams(n=m, b=1 << 12, d=d, transform="fft", seed=29)
    assert _device.compress_kernel("fft", d, 12, n1, n2, m) == 4  # SMM_KERNEL_FFT1P
    dev = P.compress_rect(torch.as_tensor(a, device="cuda"), torch.as_tensor(bm, device="cuda"), p)
    host = P.compress_rect(torch.as_tensor(a).pin_memory(), torch.as_tensor(bm), p)
    assert np.array_equal(dev.polys, host.polys)
    ref = O.compress(a, bm, b=p.b, d=d, transform="fft", seed=p.seed, threads=4)
    cf = np.linalg.norm(a @ bm)
    assert np.max(np.abs(dev.polys - ref)) <= 1e-10 * cf
    est = P.decompress_all(dev)
    est_ref, _, _ = O.decompress(ref, O.draw_words(p.seed, d, p.b), b=p.b, d=d, transform="fft", n1=n1, n2=n2,
                                 want_est=True, threads=4)
    assert np.max(np.abs(est - est_ref)) <= 1e-10 * cf


@pytest.mark.parametrize("transform", ["fwht", "fft"])
@pytest.mark.parametrize("n1,m,n2,d", [(1, 37, 5000, 3), (3000, 33, 2, 5), (8191, 41, 8192, 1), (500, 1, 700, 7),
                                       (16383, 9, 1, 3)])
def test_one_pass_edge_shapes_against_oracle(transform, n1, m, n2, d):
    """fwht1p / fft1p (b = 2^12) on ragged shapes: one-row and one-column operands, an
    inner range that is not a multiple of the 8-wide tiles, a single inner index, and
    n1 + n2 at the 16384 staging limit; against the CPU oracle (bit-exact for integer
    data, which these operands are)."""
    from oracle import sketch_oracle as O
    from paper_2601_09477_b200 import _device

    rng = np.random.default_rng(n1 * 7 + m)
    a = rng.integers(-3, 4, size=(n1, m)).astype(np.float64)
    bm = rng.integers(-3, 4, size=(m, n2)).astype(np.float64)
    p = P.SketchParams(n=m, b=1 << 12, d=d, transform=transform, seed=41)
    assert _device.compress_kernel(transform, d, 12, n1, n2, m) == (3 if transform == "fwht" else 4)
    sk = P.compress_rect(torch.as_tensor(a, device="cuda"), torch.as_tensor(bm, device="cuda"), p)
    ref = O.compress(a, bm, b=p.b, d=d, transform=transform, seed=p.seed, threads=4)
    if transform == "fwht":
        assert np.array_equal(sk.polys, ref)
    else:
        assert np.max(np.abs(sk.polys - ref)) <= 1e-10 * max(1.0, np.linalg.norm(a @ bm))


def test_extract_to_host_matches_device():
    w = W.make("cfg1", xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    sk = P.compress(w.a, w.bmat, p)
    est_d, pairs_d = P.extract_all(sk, w.threshold, strict=True)
    host = torch.empty((w.n, w.n), dtype=torch.float64).pin_memory()
    est_h, pairs_h = P.extract_all(sk, w.threshold, strict=True, est_out=host)
    assert est_h is host
    assert torch.equal(est_h, est_d.cpu())
    assert not pairs_h.is_cuda and pairs_h.is_pinned()
    assert torch.equal(pairs_h, pairs_d.cpu())
    # small row blocks exercise the 2-slot ring
    host2 = torch.empty((300, w.n), dtype=torch.float64)
    pairs2 = _device.extract_host(sk.polys_device(), sk.words, p.d, p.log2b, p.transform, w.n, w.n, 100, 400,
                                  w.threshold, True, host2, block_rows=37)
    assert torch.equal(host2, est_d[100:400].cpu())
    sel = (pairs_d[:, 0] >= 100) & (pairs_d[:, 0] < 400)
    assert torch.equal(pairs2, pairs_d[sel].cpu())


@pytest.mark.parametrize("transform,log2b,d", [("fwht", 12, 5), ("fft", 11, 3), ("fwht", 10, 9)])
def test_compress_seeds_equals_per_seed_compress(transform, log2b, d):
    # Monte-Carlo batching: stacked repetitions, one launch per <= 63
    rng = np.random.default_rng(5)
    n = 384
    a = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    b = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    p = P.SketchParams(n=n, b=1 << log2b, d=d, transform=transform, seed=0)
    seeds = list(range(100, 100 + 15))  # 15 * 9 = 135 repetitions -> three launches for d = 9
    many = P.compress_seeds(a, b, p, seeds)
    for s, sk in zip(seeds, many):
        one = P.compress(a, b, P.SketchParams(n=n, b=1 << log2b, d=d, transform=transform, seed=s))
        assert sk.hashes == one.hashes and sk.params.seed == s
        if transform == "fwht":
            assert np.array_equal(sk.polys, one.polys)
        else:
            assert np.max(np.abs(sk.polys - one.polys)) <= 1e-12 * np.max(np.abs(one.polys))
    # host operands take the streamed path
    many_h = P.compress_seeds(a.cpu(), b.cpu(), p, seeds[:3])
    for x, y in zip(many_h, many[:3]):
        assert np.max(np.abs(x.polys - y.polys)) <= 1e-12 * np.max(np.abs(y.polys))


@pytest.mark.parametrize("log2b,n1,m,n2,d", [(8, 300, 70, 200, 3), (11, 2000, 96, 1500, 3), (13, 300, 50, 300, 5),
                                             (14, 1000, 64, 900, 3), (15, 500, 40, 450, 3), (16, 700, 33, 650, 3),
                                             (18, 400, 32, 350, 3)])
def test_two_pass_fft_against_oracle(log2b, n1, m, n2, d):
    # fft2p: four-step FFT (b <= 2^14) and its frequency fold (b > 2^14), partial k-tiles,
    # rectangular operands, against the oracle (reference algorithm) at 1e-12 relative
    rng = np.random.default_rng(log2b)
    a = rng.standard_normal((n1, m))
    bm = rng.standard_normal((m, n2))
    words = O.draw_words(log2b + 100, d, 1 << log2b)
    acc = _device.compress_accumulate(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), words, d, log2b, "fft",
                                      0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    polys = _device.finalize(acc, d, log2b, "fft").cpu().numpy()
    ref = O.compress(a, bm, b=1 << log2b, d=d, words=words, transform="fft", seed=0, threads=8)
    assert np.abs(polys - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("log2b,n1,m,n2,d", [(8, 3000, 70, 2000, 3), (10, 5000, 96, 4000, 5), (12, 9000, 45, 8000, 3),
                                             (14, 1000, 1, 900, 9), (16, 700, 33, 650, 3), (17, 400, 31, 350, 3),
                                             (20, 300, 37, 280, 3),
                                             # even inner ranges: the pair mapping (b >= 2^12)
                                             (12, 9000, 46, 8000, 3), (13, 20000, 30, 300, 3), (13, 700, 34, 650, 3), (14, 3000, 62, 2000, 5),
                                             (15, 500, 2, 450, 3), (16, 900, 46, 700, 3), (18, 400, 34, 350, 3)])
def test_two_pass_fwht_against_oracle(log2b, n1, m, n2, d):
    # fwht2p across its whole range: dense pulls (n >> b: hundreds of CSR entries per warp,
    # several entry windows), a single inner index / pair, partial k-tiles, the fold (b > 2^16),
    # rectangular operands, both lane mappings; against the oracle (reference algorithm) at 1e-12 relative
    rng = np.random.default_rng(log2b + 7)
    a = rng.standard_normal((n1, m))
    bm = rng.standard_normal((m, n2))
    words = O.draw_words(log2b + 200, d, 1 << log2b)
    acc = _device.compress_accumulate(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), words, d, log2b, "fwht",
                                      0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    polys = _device.finalize(acc, d, log2b, "fwht").cpu().numpy()
    ref = O.compress(a, bm, b=1 << log2b, d=d, words=words, transform="fwht", seed=0, threads=8)
    assert np.abs(polys - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_batched_entry_queries_match_scalar_path(name):
    # per-entry queries on the device-resident sketch
    w = W.make(name, xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    sk = P.compress(w.a, w.bmat, p)
    rng = np.random.default_rng(3)
    ij = rng.integers(0, w.n, size=(500, 2))
    est, reps = P.decompress_entries(sk, ij, with_estimates=True)
    for q in range(0, 500, 25):
        i, j = int(ij[q, 0]), int(ij[q, 1])
        assert np.array_equal(reps[q], P.sketch_estimates(sk, i, j))
        assert est[q] == P.decompress_entry(sk, i, j)
    full = P.decompress_rows(sk).cpu().numpy()
    assert np.array_equal(est, full[ij[:, 0], ij[:, 1]])
    with pytest.raises(P.InvalidParameterError):
        P.decompress_entries(sk, [[0, w.n]])


@pytest.mark.parametrize("transform,log2b", [("fwht", 10), ("fwht", 17), ("fft", 10), ("fft", 15)])
def test_degenerate_hashes_everything_in_one_bucket(transform, log2b):
    # a = 0 maps every key to bucket c >> shift: one bucket holds all n inputs (the
    # gather loops' overflow paths, long CSR rows), against the oracle
    n, m = 300, 40
    rng = np.random.default_rng(11)
    a = rng.standard_normal((n, m))
    bm = rng.standard_normal((m, n))
    d = 3
    words = O.draw_words(5, d, 1 << log2b).copy()
    words[0:2 * d:2] = 0          # h1: a = 0
    words[2 * d:4 * d:2] = 0      # h2: a = 0
    acc = _device.compress_accumulate(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), words, d, log2b,
                                      transform, 0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    polys = _device.finalize(acc, d, log2b, transform).cpu().numpy()
    ref = O.compress(a, bm, b=1 << log2b, d=d, words=words, transform=transform, seed=0, threads=8)
    assert np.abs(polys - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


_PAIR_CASE = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2601_09477_b200 import _device
from oracle import sketch_oracle as O
rng = np.random.default_rng(5)
out = []
for log2b, n in ((8, 500), (10, 2000), (12, 3000), (13, 700), (14, 1024), (15, 600), (16, 1500), (17, 900)):
    a = torch.as_tensor(rng.standard_normal((n, 256)), device="cuda")
    bt = torch.as_tensor(rng.standard_normal((n + 8, 256)), device="cuda")
    words = O.draw_words(31 + log2b, 3, 1 << log2b)
    acc = _device.compress_accumulate(a, bt, words, 3, log2b, "fwht", 0, 256,
                                      a_layout=_device.KMINOR, b_layout=_device.KMINOR)
    out.append(acc.cpu().numpy())
np.savez({path!r}, *out)
"""


@pytest.mark.parametrize("_", [0])
def test_pair_mapping_bit_identical_to_one_k_per_lane(tmp_path, _):
    """The pair mapping of fwht2p (16-byte accesses, chosen automatically) and the
    one-k-per-lane mapping (SMM_NO_PAIR=1) compute the same sums in the same
    order: bit-identical accumulators on non-integer data."""
    import os
    import subprocess
    import sys

    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for tag, env in (("pair", {}), ("lane", {"SMM_NO_PAIR": "1"})):
        path = str(tmp_path / f"{tag}.npz")
        subprocess.run([sys.executable, "-c", _PAIR_CASE.format(root=root, path=path)], check=True,
                       env={**os.environ, **env}, timeout=300)
        g = np.load(path)
        res[tag] = [g[f"arr_{i}"] for i in range(len(g.files))]
    for x, y in zip(res["pair"], res["lane"]):
        assert np.array_equal(x, y)
        assert np.abs(x).max() > 0


_SLOW_CASE = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2601_09477_b200 import _device
from oracle import sketch_oracle as O
rng = np.random.default_rng(9)
out = []
for transform, log2b, n in (("fwht", 12, 700), ("fwht", 16, 900), ("fwht", 17, 500), ("fft", 12, 600),
                            ("fft", 15, 500)):
    a = torch.as_tensor(rng.standard_normal((n, 320)), device="cuda")
    bm = torch.as_tensor(rng.standard_normal((320, n)), device="cuda")
    words = O.draw_words(7 + log2b, 3, 1 << log2b)
    acc = _device.compress_accumulate(a, bm, words, 3, log2b, transform, 0, 320, a_layout=_device.KMINOR)
    out.append(acc.cpu().numpy())
    # accumulate mode: two calls over [0, 160) and [160, 320) continue one k order
    acc2 = _device.compress_accumulate(a[:, :160], bm[:160], words, 3, log2b, transform, 0, 160,
                                       a_layout=_device.KMINOR)
    _device.compress_accumulate(a[:, 160:], bm[160:], words, 3, log2b, transform, 0, 160, acc=acc2,
                                a_layout=_device.KMINOR, accumulate=True)
    out.append(acc2.cpu().numpy())
np.savez({path!r}, *out)
"""


def test_accumulator_slow_path_bit_identical(tmp_path):
    """SMM_ACC_SLOWPATH=1 sends every pass-2 item of fwht2p / fft2p through the
    accumulator slow path (per-warp acquire of the slice counter at the end of the
    item instead of the scheduler's acquire before it): same k order, so the
    accumulators must be bit-identical to the default run, in one call and in
    accumulate mode across two calls."""
    import os
    import subprocess
    import sys

    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for tag, env in (("fast", {}), ("slow", {"SMM_ACC_SLOWPATH": "1"})):
        path = str(tmp_path / f"{tag}.npz")
        subprocess.run([sys.executable, "-c", _SLOW_CASE.format(root=root, path=path)], check=True,
                       env={**os.environ, **env}, timeout=300)
        g = np.load(path)
        res[tag] = [g[f"arr_{i}"] for i in range(len(g.files))]
    for i, (x, y) in enumerate(zip(res["fast"], res["slow"])):
        assert np.array_equal(x, y), i
        assert np.abs(x).max() > 0
    # one call and two accumulate-mode calls agree as well (FWHT two-pass: bit for bit)
    for i in (0, 2, 4):
        assert np.array_equal(res["fast"][i], res["fast"][i + 1]), i



@pytest.mark.parametrize("transform", ["fwht", "fft"])
def test_compress_seeds_stacked_against_oracle(transform):
    """Three seeds stacked into one launch (compress_seeds) against the CPU oracle of
    each seed separately (the reference's Monte-Carlo drivers call compress once per
    seed, experiments.py:216-312)."""
    rng = np.random.default_rng(41)
    n = 384
    a, m = rng.normal(size=(n, n)), rng.normal(size=(n, n))
    p = P.SketchParams(n=n, b=1 << 12, d=5, transform=transform, seed=1)
    seeds = [101, 202, 303]
    sks = P.compress_seeds(a, m, p, seeds)
    cn = _cnorm(a, m)
    for sk, seed in zip(sks, seeds):
        ref = O.compress(a, m, b=p.b, d=p.d, transform=transform, seed=seed, threads=8)
        assert sk.params.seed == seed
        assert np.max(np.abs(sk.polys - ref)) <= TOL * cn
        eref, _, _ = O.decompress(ref, O.draw_words(seed, p.d, p.b), b=p.b, d=p.d, transform=transform, n1=n, n2=n)
        assert np.max(np.abs(P.decompress_all(sk) - eref)) <= TOL * cn


@pytest.mark.parametrize("transform,d,b", [("fwht", 65, 1 << 10), ("fft", 65, 1 << 9), ("fwht", 129, 1 << 12),
                                           ("fft", 101, 1 << 12)])
def test_depth_beyond_one_launch_against_oracle(transform, d, b):
    """d > 63 (the reference accepts any odd d, sketch.py:75-76): compress runs in
    repetition groups of 63, extraction / queries / heavy hitters read the hash
    functions from device memory; all against the CPU oracle."""
    rng = np.random.default_rng(d)
    n = 160
    a, m = rng.normal(size=(n, n)), rng.normal(size=(n, n))
    p = P.SketchParams(n=n, b=b, d=d, transform=transform, seed=77)
    sk = P.compress(a, m, p)
    ref = O.compress(a, m, b=b, d=d, transform=transform, seed=77, threads=8)
    cn = _cnorm(a, m)
    assert sk.polys.shape == (d, b)
    assert np.max(np.abs(sk.polys - ref)) <= TOL * cn
    words = O.draw_words(77, d, b)
    thr = 0.25 * float(np.abs(a @ m).max())
    eref, cnt, hh_ref = O.decompress(ref, words, b=b, d=d, transform=transform, n1=n, n2=n, thr=thr, strict=True,
                                     want_hh=True)
    est = P.decompress_all(sk)
    assert np.max(np.abs(est - eref)) <= TOL * cn
    hh = P.heavy_hitters(sk, thr, strict=True)
    assert np.array_equal(hh, np.argwhere(np.abs(est) > thr))
    ij = np.array([[0, 0], [5, 17], [n - 1, n - 1], [80, 3]])
    q = P.decompress_entries(sk, ij)
    assert np.array_equal(np.asarray(q), est[ij[:, 0], ij[:, 1]])
    # the hash tables of every repetition (groups of 63 launches) against the oracle
    h1, s1, _, _ = O.tables(words, d, b, n, n)
    assert np.array_equal(_device.hash_table(sk.hashes, 0, n).cpu().numpy().astype(np.int64), h1)
    assert np.array_equal(_device.hash_table(sk.hashes, 2, n).cpu().numpy().astype(np.float64), s1)


@pytest.mark.parametrize("transform", ["fwht", "fft"])
@pytest.mark.parametrize("n", [40, 3000, 12000])
def test_degenerate_bucket_keeps_the_reference_order(transform, n):
    """Every input in one bucket (hash a = 0): the CSR fill is atomic, the segmented
    sort (one thread up to 32 entries, a CTA bitonic network in shared memory up to
    8192, in global memory beyond) must restore increasing input order — the
    reference's serial scatter order (sketch.py:166-172).  With two inner indices the
    sketch is bit-identical to the oracle only if the bucket sums are added in that
    order."""
    rng = np.random.default_rng(n)
    m, d, log2b = 2, 3, 10
    a = rng.standard_normal((n, m))
    bm = rng.standard_normal((m, n))
    words = O.draw_words(5, d, 1 << log2b).copy()
    words[0:2 * d:2] = 0          # h1: a = 0
    words[2 * d:4 * d:2] = 0      # h2: a = 0
    acc = _device.compress_accumulate(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), words, d, log2b,
                                      transform, 0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    polys = _device.finalize(acc, d, log2b, transform).cpu().numpy()
    ref = O.compress(a, bm, b=1 << log2b, d=d, words=words, transform=transform, seed=0, threads=1)
    if transform == "fwht":
        assert np.array_equal(polys, ref)
    else:
        assert np.abs(polys - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())
