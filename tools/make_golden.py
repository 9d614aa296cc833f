"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/make_golden.py [small|configs|cfg4|cfg5|all]

Outputs go to tests/golden/ and are committed.  Nothing here is imported by
the product package or by the GPU tests at run time; tests read the fixtures.

Fixture provenance:
  * hash_golden.json   reference eval_bucket/eval_sign on the golden pairs pinned
                       by the reference's own tests (frontend/tests/hash.test.ts:16-36,
                       tests/test_hashing.py:62-73); the TS expected values are
                       parsed from the test file and cross-checked here.
  * draws.json         reference SketchHashes.draw packed words (hashing.py:123-152)
  * small_cases.npz    reference compress/compress_rect/decompress_all on seeded
                       small inputs (edge cases included), threads 1 and 3
  * transforms.json    reference fwht_inplace / xor_convolve / fft_forward /
                       fft_inverse / cyclic_convolve known answers
  * containers.npz     reference sketch_to_bytes for two sketches
  * cfg*.npz           reference runs on the BASELINE configs (workloads.py)
"""

from __future__ import annotations

import hashlib
import json
import re
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tests" / "golden"
REF_TS = Path("/root/reference/pkg/frontend/tests/hash.test.ts")

import sketchmm as S  # noqa: E402  (the reference)
from sketchmm import hashing as RH  # noqa: E402
from sketchmm import sketch as RS  # noqa: E402
from sketchmm import transforms as RT  # noqa: E402

from paper_2601_09477_b200 import workloads as W  # noqa: E402


def _versions():
    import numba
    return {"numpy": np.__version__, "numba": numba.__version__}


def hash_golden():
    src = REF_TS.read_text()
    keys = [int(x) for x in re.search(r"const KEYS = \[([^\]]*)\]", src).group(1).split(",")]
    entries = []
    for m in re.finditer(r"pair: \{ a: ([^,]+), c: ([^,]+), shift: (\d+) \},\s*buckets: \[([^\]]*)\],\s*signs: \[([^\]]*)\]", src):
        def big(s):
            s = s.strip()
            mm = re.fullmatch(r"1n << (\d+)n", s)
            if mm:
                return 1 << int(mm.group(1))
            return int(s.rstrip("n"), 0)
        a, c, shift = big(m.group(1)), big(m.group(2)), int(m.group(3))
        buckets = [int(x) for x in m.group(4).split(",")]
        signs = [int(x) for x in m.group(5).split(",")]
        ref_b = [RH.eval_bucket(RH.HashPair(a=a, c=c, shift=shift), x) for x in keys]
        ref_s = [RH.eval_sign(RH.HashPair(a=a, c=c, shift=63), x) for x in keys]
        assert ref_b == buckets and ref_s == signs, "reference disagrees with the TS golden vectors"
        entries.append({"a": str(a), "c": str(c), "shift": shift, "keys": keys, "buckets": buckets, "signs": signs})
    # test_hashing.py:62-73 known values and the wrap-around cases of hash.test.ts:45-51
    extra = [
        (2**62, 0, 62, 1), (1, 2**63, 63, 0), (2**63, 0, 63, 2), ((1 << 64) - 1, 0, 62, 1), ((1 << 64) - 1, 0, 62, 3),
    ]
    known = []
    for a, c, shift, x in extra:
        known.append({"a": str(a), "c": str(c), "shift": shift, "x": x,
                      "bucket": RH.eval_bucket(RH.HashPair(a=a, c=c, shift=shift), x),
                      "sign": RH.eval_sign(RH.HashPair(a=a, c=c, shift=63), x)})
    # a denser random table for the device hash-table kernel (bit-exact contract)
    rng = np.random.default_rng(2024)
    tables = []
    for shift in (32, 44, 48, 50, 52, 54, 58, 62, 63):
        a, c = (int(v) for v in rng.integers(0, 1 << 64, size=2, dtype=np.uint64))
        xs = np.arange(2000, dtype=np.uint64)
        tables.append({"a": str(a), "c": str(c), "shift": shift,
                       "buckets": RH.bucket_many(RH.HashPair(a=a, c=c, shift=shift), xs).tolist(),
                       "signs": RH.sign_many(RH.HashPair(a=a, c=c, shift=63), xs).astype(int).tolist()})
    (OUT / "hash_golden.json").write_text(json.dumps({"ts_vectors": entries, "known": known, "tables": tables,
                                                      "versions": _versions()}, indent=1))


def draws():
    out = []
    for seed in (0, 1, 5, 7, 12, 77, 201, 202, 203, 204, 205, 2**64 - 1):
        for d in (1, 3, 5, 7, 9):
            for b in (2, 16, 4096, 1 << 16, 1 << 20, 1 << 32):
                h = RH.SketchHashes.draw(np.random.default_rng(seed), d, b)
                out.append({"seed": str(seed), "d": d, "b": b, "words": [str(int(w)) for w in h.packed_words()],
                            "digest": h.digest()})
    (OUT / "draws.json").write_text(json.dumps({"draws": out, "versions": _versions()}))


def _case(rng, name, transform, n1, m, n2, b, d, seed, threads, kind="normal"):
    if kind == "zeros":
        a = np.zeros((n1, m))
        bm = np.zeros((m, n2))
    elif kind == "ints":
        a = rng.integers(-3, 4, size=(n1, m)).astype(np.float64)
        bm = rng.integers(-3, 4, size=(m, n2)).astype(np.float64)
    else:
        a = rng.normal(size=(n1, m))
        bm = rng.normal(size=(m, n2))
    p = RS.SketchParams(n=m, b=b, d=d, transform=transform, seed=seed)
    sk = RS.compress_rect(a, bm, p, threads=threads) if (n1 != m or n2 != m) else RS.compress(a, bm, p, threads=threads)
    est = RS.decompress_all(sk)
    return {f"{name}/a": a, f"{name}/b": bm, f"{name}/polys": sk.polys, f"{name}/est": est,
            f"{name}/words": sk.hashes.packed_words(),
            f"{name}/meta": np.array([n1, m, n2, b, d, seed, threads, 1 if transform == "fwht" else 0], dtype=np.int64)}


def small_cases():
    rng = np.random.default_rng(7)
    arrays = {}
    names = []
    specs = []
    for transform in ("fwht", "fft"):
        for b in (2, 4, 16, 64, 256, 1024):
            for d in (1, 3, 5):
                specs.append((transform, 16, 16, 16, b, d, 77, 1, "normal"))
        specs += [
            (transform, 1, 1, 1, 2, 1, 3, 1, "normal"),
            (transform, 6, 8, 10, 16, 3, 21, 1, "normal"),  # rectangular (test_sketch.py:241-255)
            (transform, 8, 8, 8, 16, 3, 1, 1, "zeros"),
            (transform, 32, 32, 32, 64, 3, 15, 3, "normal"),  # chunked (threads=3)
            (transform, 64, 64, 64, 32, 5, 9, 2, "ints"),  # b < n, integer-valued
            (transform, 64, 64, 64, 512, 7, 7, 1, "normal"),
            (transform, 100, 40, 70, 128, 3, 11, 1, "normal"),  # non power-of-two shapes
            (transform, 4, 4, 4, 16, 1, {"fwht": 5, "fft": 12}[transform], 1, "normal"),  # INJECTIVE_SEED
        ]
    for q, (transform, n1, m, n2, b, d, seed, th, kind) in enumerate(specs):
        name = f"c{q:03d}_{transform}_{n1}x{m}x{n2}_b{b}_d{d}_{kind}"
        arrays.update(_case(rng, name, transform, n1, m, n2, b, d, seed, th, kind))
        names.append(name)
    np.savez_compressed(OUT / "small_cases.npz", names=np.array(names), **arrays)


def transforms_golden():
    rng = np.random.default_rng(42)
    out = {}
    out["fwht_1234"] = RT.fwht_inplace(np.array([1.0, 2, 3, 4])).tolist()
    out["fwht_impulse"] = RT.fwht_inplace(np.array([1.0, 0, 0, 0])).tolist()
    out["xor_12_34"] = RT.xor_convolve([1, 2], [3, 4]).tolist()
    out["cyc_12_34"] = RT.cyclic_convolve([1, 2], [3, 4]).tolist()
    z = RT.fft_forward([0, 1, 0, 0])
    out["fft_0100"] = [[v.real, v.imag] for v in z]
    vecs = {}
    for b in (2, 8, 64, 1024, 4096):
        x = rng.normal(size=b)
        y = rng.normal(size=b)
        vecs[str(b)] = {"x": x.tolist(), "y": y.tolist(), "fwht": RT.fwht_inplace(x.copy()).tolist(),
                        "xor": RT.xor_convolve(x, y).tolist(), "cyc": RT.cyclic_convolve(x, y).tolist(),
                        "fft_re": RT.fft_forward(x).real.tolist(), "fft_im": RT.fft_forward(x).imag.tolist()}
    out["vectors"] = vecs
    (OUT / "transforms.json").write_text(json.dumps(out))


def containers():
    rng = np.random.default_rng(17)
    arrays = {}
    for transform in ("fwht", "fft"):
        a = rng.normal(size=(8, 8))
        m = rng.normal(size=(8, 8))
        sk = RS.compress(a, m, RS.SketchParams(n=8, b=16, d=3, transform=transform, seed=18), threads=1)
        arrays[f"{transform}/a"] = a
        arrays[f"{transform}/b"] = m
        arrays[f"{transform}/bytes"] = np.frombuffer(RS.sketch_to_bytes(sk), dtype=np.uint8)
    np.savez_compressed(OUT / "containers.npz", **arrays)


def _sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def config_golden(name: str, threads: int = 8, full_polys: bool = False, sample: int = 4096):
    t0 = time.time()
    w = W.make(name)
    p = RS.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    tc = time.perf_counter()
    sk = RS.compress(w.a, w.bmat, p, threads=threads)
    tc = time.perf_counter() - tc
    td = time.perf_counter()
    est = RS.decompress_all(sk)
    td = time.perf_counter() - td
    ab = np.abs(est)
    hh_mask = ab > w.threshold if w.strict else ab >= w.threshold
    hh = np.argwhere(hh_mask).astype(np.int64)
    rng = np.random.default_rng(99)
    si = rng.integers(0, w.n, size=sample)
    sj = rng.integers(0, w.n, size=sample)
    cnorm = float(np.sqrt(np.sum((w.a @ w.bmat) ** 2))) if w.n <= 8192 else float("nan")
    arrays = {
        "words": sk.hashes.packed_words(),
        "polys_sha256": np.frombuffer(_sha(sk.polys).encode(), dtype=np.uint8),
        "polys_rowsum": sk.polys.sum(axis=1),
        "polys_sample_idx": rng.integers(0, w.b, size=(w.d, 1024)),
        "est_sample_ij": np.stack([si, sj], axis=1),
        "est_sample": est[si, sj],
        "est_big": est[w.big[:, 0], w.big[:, 1]] if w.big.size else np.zeros(0),
        "hh_count": np.array([hh.shape[0]]),
        "hh_sha256": np.frombuffer(_sha(hh).encode(), dtype=np.uint8),
        "est_rowsum": est.sum(axis=1),
        "meta": np.array([w.n, w.b, w.d, threads], dtype=np.int64),
        "cnorm": np.array([cnorm]),
        "timing_s": np.array([tc, td]),
    }
    arrays["polys_sample"] = np.take_along_axis(sk.polys, arrays["polys_sample_idx"], axis=1)
    if full_polys:
        arrays["polys"] = sk.polys
    if hh.shape[0] <= 200000:
        arrays["hh"] = hh
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"{name}: compress {tc:.1f}s decompress {td:.1f}s hh={hh.shape[0]} total {time.time() - t0:.1f}s", flush=True)


def matrix_files():
    """Matrix files written by the reference's matio (cli.py multiply's I/O)."""
    from sketchmm import matio

    m = np.array([[1.0, -2.5, 3.0e-300, 0.1], [np.pi, -0.0, 1e300, 7.0], [2.0 ** -1074, 5.0, -6.0, 1.0 / 3.0]])
    matio.save_matrix_binary(OUT / "matrix_ref.dmat", m)
    matio.save_matrix_csv(OUT / "matrix_ref.csv", m)
    np.save(OUT / "matrix_ref.npy", m)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    OUT.mkdir(parents=True, exist_ok=True)
    if what in ("small", "all"):
        hash_golden()
        draws()
        small_cases()
        transforms_golden()
        containers()
        print("small fixtures written")
    if what in ("configs", "all"):
        config_golden("cfg1", full_polys=True)
        config_golden("cfg2", full_polys=True)
        config_golden("cfg3", full_polys=False)
    if what in ("cfg4", "all"):
        config_golden("cfg4", full_polys=False)
    if what in ("cfg5", "all"):
        for nnz in W.CFG5_NNZ:
            for transform in ("fwht", "fft"):
                for b in W.CFG5_B[:3]:
                    for d in W.CFG5_D:
                        config_golden(W.cfg5_name(b, d, nnz, transform), full_polys=(b <= 1 << 14 and nnz == 512))
    if what in ("matrix", "all"):
        matrix_files()
    if what == "cfg5rest":  # every remaining cfg5 point (b = 2^18, 2^20), skipping existing fixtures
        for b in W.CFG5_B[3:]:
            for d in W.CFG5_D:
                for nnz in W.CFG5_NNZ:
                    for transform in ("fwht", "fft"):
                        name = W.cfg5_name(b, d, nnz, transform)
                        if not (OUT / f"{name}.npz").exists():
                            config_golden(name)
    if what == "cfg5big":
        for transform in ("fwht", "fft"):
            for b in W.CFG5_B[3:]:
                config_golden(W.cfg5_name(b, 3, 512, transform))


if __name__ == "__main__":
    main()
