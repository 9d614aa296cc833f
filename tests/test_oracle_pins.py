"""Pin the CPU oracle to the reference's own outputs (CPU-only).

The fixtures in tests/golden/ were produced by running the reference package
itself (tools/make_golden.py).  The C oracle must reproduce them bit for bit at
the same chunk count; the pure-numpy ``compress_slow`` must agree within the
reference's own 1e-9 bound (reference tests/test_sketch.py:100-109).
"""

import hashlib

import numpy as np
import pytest

from conftest import cfg_golden
from oracle import sketch_oracle as O


def test_oracle_small_cases_bit_exact(small_cases):
    for c in small_cases:
        words = O.draw_words(c["seed"], c["d"], c["b"])
        assert np.array_equal(words, c["words"]), c["name"]
        pretrans = False
        polys = O.compress(c["a"], c["bm"], b=c["b"], d=c["d"], transform=c["transform"], seed=c["seed"],
                           threads=c["threads"], pretransposed=pretrans)
        assert np.array_equal(polys, c["polys"]), c["name"]
        est, _, _ = O.decompress(c["polys"], words, b=c["b"], d=c["d"], transform=c["transform"],
                                 n1=c["n1"], n2=c["n2"])
        assert np.array_equal(est, c["est"]), c["name"]


def test_compress_slow_matches_reference(small_cases):
    # reference test_sketch.py:100-109: |fast - slow| < 1e-9 * max(1, |slow|max)
    for c in small_cases:
        if c["b"] > 256 or c["m"] > 32:
            continue
        slow = O.compress_slow(c["a"], c["bm"], b=c["b"], d=c["d"], transform=c["transform"], seed=c["seed"])
        scale = max(1.0, np.abs(slow).max())
        assert np.max(np.abs(c["polys"] - slow)) < 1e-9 * scale, c["name"]


def test_hash_words_match_reference_draws(draws_golden):
    for e in draws_golden:
        words = O.draw_words(int(e["seed"]), e["d"], e["b"])
        assert [str(int(w)) for w in words] == e["words"]


def test_hash_tables_match_golden(hash_golden):
    for tab in hash_golden["tables"]:
        a, c, shift = int(tab["a"]), int(tab["c"]), tab["shift"]
        b = 1 << (64 - shift)
        words = np.array([a, c, a, c, a, c, a, c], dtype=np.uint64)
        h = O.bucket_table(words, 1, b, 0, 2000)[0]
        s = O.sign_table(words, 1, 2, 2000)[0]
        assert h.tolist() == tab["buckets"]
        assert s.astype(int).tolist() == tab["signs"]


def test_transform_known_answers(transforms_golden):
    g = transforms_golden
    assert O.fwht(np.array([1.0, 2, 3, 4])).tolist() == g["fwht_1234"] == [10, -2, -4, 0]
    assert O.fwht(np.array([1.0, 0, 0, 0])).tolist() == g["fwht_impulse"]
    z = O.fft_forward_half(np.array([0.0, 1, 0, 0]))
    assert np.allclose(z, [complex(*v) for v in g["fft_0100"]], atol=1e-12)
    for b, v in g["vectors"].items():
        x = np.array(v["x"])
        assert np.array_equal(O.fwht(x), np.array(v["fwht"]))
        zz = O.fft_forward_half(x)
        assert np.array_equal(zz.real, np.array(v["fft_re"])) and np.array_equal(zz.imag, np.array(v["fft_im"]))


@pytest.mark.parametrize("name", ["cfg1"])
def test_oracle_matches_reference_on_config(name):
    from paper_2601_09477_b200 import workloads as W

    g = cfg_golden(name)
    w = W.make(name)
    threads = int(g["meta"][3])
    polys = O.compress(w.a, w.bmat, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed, threads=threads)
    assert np.array_equal(polys, g["polys"])
    assert hashlib.sha256(polys.tobytes()).hexdigest() == bytes(g["polys_sha256"]).decode()
    _, cnt, hh = O.decompress(polys, g["words"], b=w.b, d=w.d, transform=w.transform, n1=w.n, n2=w.n,
                              thr=w.threshold, strict=True, want_est=False, want_hh=True)
    assert cnt == int(g["hh_count"][0])
    assert hashlib.sha256(np.ascontiguousarray(hh).tobytes()).hexdigest() == bytes(g["hh_sha256"]).decode()


def test_accumulate_is_additive_over_k_ranges():
    # the k-shard unit: acc[0,m) == acc[0,k) + acc[k,m) exactly for integer data
    rng = np.random.default_rng(3)
    n, b, d = 48, 64, 3
    a = rng.integers(-2, 3, size=(n, n)).astype(np.float64)
    bm = rng.integers(-2, 3, size=(n, n)).astype(np.float64)
    words = O.draw_words(5, d, b)
    at = np.ascontiguousarray(a.T)
    full = O.accumulate_fwht(at, bm, b=b, d=d, words=words, k0=0, k1=n)
    parts = O.accumulate_fwht(at, bm, b=b, d=d, words=words, k0=0, k1=17) + \
        O.accumulate_fwht(at, bm, b=b, d=d, words=words, k0=17, k1=n)
    assert np.array_equal(full, parts)
    polys = O.fwht_inverse_scaled(full)
    ref = O.compress(a, bm, b=b, d=d, transform="fwht", seed=5, threads=1)
    assert np.array_equal(polys, ref)


def test_oracle_median_propagates_nan_like_numpy():
    # sketch.py:398 takes np.median over the d values: one NaN among them gives NaN
    n, b, d = 16, 32, 3
    words = O.draw_words(4, d, b)
    polys = np.random.default_rng(1).normal(size=(d, b))
    polys[1, 7] = np.nan
    est, cnt, _ = O.decompress(polys, words, b=b, d=d, transform="fwht", n1=n, n2=n, thr=0.0, strict=True)
    h1, s1, h2, s2 = O.tables(words, d, b, n, n)
    vals = np.stack([polys[t][h1[t][:, None] ^ h2[t][None, :]] * s1[t][:, None] * s2[t][None, :] for t in range(d)])
    want = np.median(vals, axis=0)
    assert np.array_equal(np.isnan(est), np.isnan(want)) and np.isnan(est).any()
    ok = ~np.isnan(want)
    assert np.array_equal(est[ok], want[ok])
    assert int(cnt) == int(np.sum(np.abs(want[ok]) > 0.0))
