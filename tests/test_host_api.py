"""Host-side API contract (CPU-only): parameters, hash drawing, containers and
the C-ABI library surface.  Mirrors the reference's own unit tests
(tests/test_sketch.py TestParams / TestSerialization, tests/test_hashing.py)."""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2601_09477_b200 as P
from paper_2601_09477_b200 import _lib
from paper_2601_09477_b200.errors import FormatError, InvalidParameterError
from paper_2601_09477_b200.hashing import HashPair, SketchHashes, draw_hash, eval_bucket, eval_sign

ROOT = Path(__file__).resolve().parents[1]


class TestParams:
    def test_valid(self):
        p = P.SketchParams(n=16, b=64, d=3, transform="fft", seed=9)
        assert (p.n, p.b, p.d, p.log2b) == (16, 64, 3, 6)

    @pytest.mark.parametrize("kw", [dict(n=0, b=16, d=1), dict(n=8, b=24, d=1), dict(n=8, b=1, d=1),
                                    dict(n=8, b=2**33, d=1), dict(n=8, b=16, d=2), dict(n=8, b=16, d=0),
                                    dict(n=8, b=16, d=1, transform="dct"), dict(n=8, b=16, d=1, seed=-1)])
    def test_invalid(self, kw):
        with pytest.raises(InvalidParameterError):
            P.SketchParams(**{"transform": "fwht", "seed": 0, **kw})

    def test_derive(self):
        p = P.derive_params(1024, 1.0, 0.5)
        assert p.d == 11 and p.b == 512
        assert P.derive_params(2**15, 0.25, 1.0).d == 3
        assert P.derive_params(1024, 1.5, 4.0).d == 15
        for bad in [(1024, 1.0, 0.3), (1024, 1.0, 3.0), (1000, 1.0, 1.0), (1024, -1.0, 1.0)]:
            with pytest.raises(InvalidParameterError):
                P.derive_params(*bad)

    def test_effective_threads(self):
        assert P.effective_threads(3) == 3
        with pytest.raises(InvalidParameterError):
            P.effective_threads(0)

    def test_invalid_parameter_is_value_error(self):
        assert issubclass(InvalidParameterError, ValueError)


class TestHashing:
    def test_draw_matches_reference_words(self, draws_golden):
        for e in draws_golden:
            h = SketchHashes.draw(np.random.default_rng(int(e["seed"])), e["d"], e["b"])
            assert [str(int(w)) for w in h.packed_words()] == e["words"]
            assert h.digest() == e["digest"]

    def test_ts_golden_vectors(self, hash_golden):
        # reference frontend/tests/hash.test.ts:16-36 (cross-checked against the reference)
        for e in hash_golden["ts_vectors"]:
            a, c, shift = int(e["a"]), int(e["c"]), e["shift"]
            assert [eval_bucket(HashPair(a, c, shift), x) for x in e["keys"]] == e["buckets"]
            assert [eval_sign(HashPair(a, c, 63), x) for x in e["keys"]] == e["signs"]
        for k in hash_golden["known"]:
            assert eval_bucket(HashPair(int(k["a"]), int(k["c"]), k["shift"]), k["x"]) == k["bucket"]

    def test_shift_and_validation(self):
        assert draw_hash(np.random.default_rng(1), 2).shift == 63
        assert draw_hash(np.random.default_rng(1), 2**32).shift == 32
        for b in (0, 1, 3, 100, 2**33):
            with pytest.raises(InvalidParameterError):
                draw_hash(np.random.default_rng(0), b)
        with pytest.raises(InvalidParameterError):
            HashPair(a=2**64, c=0, shift=60)
        with pytest.raises(InvalidParameterError):
            HashPair(a=0, c=0, shift=20)

    def test_cached_draw_equals_reference_draw(self, draws_golden):
        # compress reuses the draw per (seed, d, b) (sketch._drawn): same words as a fresh
        # default_rng(seed) draw, and the shared words cannot be modified in place
        from paper_2601_09477_b200.sketch import _drawn

        for e in draws_golden[:40]:
            for _ in range(2):
                h, w = _drawn(int(e["seed"]), e["d"], e["b"])
                assert [str(int(x)) for x in w] == e["words"]
                assert h == SketchHashes.draw(np.random.default_rng(int(e["seed"])), e["d"], e["b"])
                assert not w.flags.writeable

    def test_json_round_trip(self):
        g = SketchHashes.draw(np.random.default_rng(3), 5, 256)
        assert SketchHashes.from_json_obj(json.loads(json.dumps(g.to_json_obj()))) == g
        assert SketchHashes.from_words(g.packed_words(), 5, 256) == g


class TestContainer:
    def test_reference_bytes_round_trip(self, golden_dir):
        g = np.load(golden_dir / "containers.npz")
        for tr in ("fwht", "fft"):
            raw = g[f"{tr}/bytes"].tobytes()
            sk = P.sketch_from_bytes(raw)
            assert sk.params.transform == tr and sk.params.n == 8 and sk.params.d == 3
            assert P.sketch_to_bytes(sk) == raw  # byte-for-byte with the reference writer

    def test_malformed(self, golden_dir):
        raw = np.load(golden_dir / "containers.npz")["fwht/bytes"].tobytes()
        for bad in (b"JUNK" + raw[4:], raw[:-1], raw[:20]):
            with pytest.raises(FormatError):
                P.sketch_from_bytes(bad)
        v = bytearray(raw)
        v[4] = 9
        with pytest.raises(FormatError):
            P.sketch_from_bytes(bytes(v))

    def test_header_layout(self, golden_dir):
        raw = np.load(golden_dir / "containers.npz")["fwht/bytes"].tobytes()
        assert raw[:4] == b"SKCH" and len(raw) == 44 + 8 * 8 * 3 + 8 * 3 * 16

    def test_rectangular_not_serializable(self):
        h = SketchHashes.draw(np.random.default_rng(0), 1, 16)
        sk = P.ProductSketch(np.zeros((1, 16)), h, P.SketchParams(n=8, b=16, d=1), 4, 6)
        with pytest.raises(InvalidParameterError):
            P.sketch_to_bytes(sk)


def test_workspace_estimate_monotone():
    assert 0 < P.estimate_workspace_bytes(64, 256, 3, "fwht", 1) < P.estimate_workspace_bytes(1024, 4096, 15, "fwht", 1)


# ------------------------------------------------------------------ C ABI surface
def _header_symbols():
    text = (ROOT / "include" / "sketchmm_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char \*)\s*(smm_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.smm_abi_version() == 1


def test_abi_rejects_bad_parameters_before_any_kernel():
    lib = _lib.load()
    words = np.zeros(8 * 3, dtype=np.uint64)
    wp = words.ctypes.data_as(ctypes.c_void_p)
    out = ctypes.c_int64(0)
    # depth out of range, zero width, bad variant -> SMM_ERR_INVALID (maps to InvalidParameterError);
    # compress accepts even depths (stacked seeds, compress_seeds), extraction does not
    assert lib.smm_compress_workspace(1, 0, 4, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_ERR_INVALID
    assert lib.smm_compress_workspace(1, _lib.MAX_DEPTH_TOTAL + 1, 4, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_ERR_INVALID
    # deeper than one launch (groups of 63 repetitions): accepted, same workspace as one group
    w63, w65 = ctypes.c_int64(0), ctypes.c_int64(0)
    assert lib.smm_compress_workspace(1, 63, 12, 64, 64, 0, 64, ctypes.byref(w63)) == _lib.SMM_OK
    assert lib.smm_compress_workspace(1, 65, 12, 64, 64, 0, 64, ctypes.byref(w65)) == _lib.SMM_OK
    assert w63.value == w65.value > 0
    # extraction past 63 repetitions carries the hash functions in its workspace
    assert lib.smm_extract_workspace(63, 8, 8, 0, 8, ctypes.byref(w63)) == _lib.SMM_OK
    assert lib.smm_extract_workspace(65, 8, 8, 0, 8, ctypes.byref(w65)) == _lib.SMM_OK
    assert w65.value >= w63.value + 65 * 64
    assert lib.smm_compress_workspace(1, 2, 4, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_OK
    assert lib.smm_extract(1, None, wp, 2, 4, 8, 8, 0, 8, None, 8, 0.5, 1, None, 0, None, None, 0,
                           None) == _lib.SMM_ERR_INVALID
    assert b"odd" in lib.smm_last_error()
    assert lib.smm_compress_workspace(1, 3, 0, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_ERR_INVALID
    assert lib.smm_compress_workspace(7, 3, 4, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_ERR_INVALID
    rc = lib.smm_compress_accumulate(1, None, 8, None, 8, 8, 8, 4, 2, wp, 3, 4, None, None, 0, None)
    assert rc == _lib.SMM_ERR_INVALID
    with pytest.raises(InvalidParameterError):
        _lib.check(rc)
    assert b"NULL" in lib.smm_last_error() or b"range" in lib.smm_last_error()
    assert lib.smm_extract_workspace(3, 8, 8, 4, 9, ctypes.byref(out)) == _lib.SMM_ERR_INVALID
    assert lib.smm_compress_workspace(1, 3, 4, 8, 8, 0, 8, ctypes.byref(out)) == _lib.SMM_OK and out.value > 0
    # live kernel timing: nothing recorded yet, bad channel rejected
    tot, cnt = ctypes.c_double(-1.0), ctypes.c_int64(-1)
    assert lib.smm_kernel_timing(0) == _lib.SMM_OK
    assert lib.smm_kernel_timing_read(0, ctypes.byref(tot), ctypes.byref(cnt)) == _lib.SMM_OK
    assert tot.value == 0.0 and cnt.value == 0
    assert lib.smm_kernel_timing_read(2, ctypes.byref(tot), ctypes.byref(cnt)) == _lib.SMM_ERR_INVALID


def test_api_validates_before_device_work():
    p = P.SketchParams(n=8, b=16, d=1)
    # shape violations raise InvalidParameterError even without a GPU (reference sketch.py:298-301)
    import torch

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    with pytest.raises(InvalidParameterError):
        P.compress(np.zeros((8, 8)), np.zeros((4, 4)), p)
    with pytest.raises(InvalidParameterError):
        P.compress(np.zeros(8), np.zeros((8, 8)), p)
    with pytest.raises(InvalidParameterError):
        P.compress_rect(np.zeros((4, 6)), np.zeros((6, 4)), p)
    with pytest.raises(InvalidParameterError):
        P.compress(np.zeros((8, 8)), np.zeros((8, 8)), p, threads=0)
    # valid input without a GPU fails loudly: there is no CPU fallback
    with pytest.raises(RuntimeError):
        P.compress(np.zeros((8, 8)), np.zeros((8, 8)), p)


def test_compress_kernel_family_dispatch():
    """smm_compress_kernel: which kernel family serves a shape (compress_seeds stacks
    seeds only within one family, so every sketch keeps its single-call bits)."""
    from paper_2601_09477_b200 import _device

    K = {"fold": 0, "fwht2p": 1, "fft2p": 2, "fwht1p": 3, "fft1p": 4}
    assert _device.compress_kernel("fwht", 3, 12, 8192, 8192, 8192) == K["fwht1p"]   # cfg5 b = 2^12
    assert _device.compress_kernel("fwht", 3, 12, 1024, 1024, 1024) == K["fwht1p"]   # cfg1
    assert _device.compress_kernel("fwht", 9, 12, 8192, 8192, 8192) == K["fwht1p"]   # d > 7: repetition groups
    assert _device.compress_kernel("fwht", 63, 12, 8192, 8192, 8192) == K["fwht1p"]
    assert _device.compress_kernel("fwht", 3, 12, 16384, 16384, 16384) == K["fwht2p"]  # columns exceed smem
    assert _device.compress_kernel("fwht", 5, 16, 16384, 16384, 16384) == K["fwht2p"]  # cfg3
    assert _device.compress_kernel("fft", 5, 14, 4096, 4096, 4096) == K["fft2p"]     # cfg2
    assert _device.compress_kernel("fft", 5, 12, 8192, 8192, 8192) == K["fft1p"]     # cfg5 b = 2^12 FFT
    assert _device.compress_kernel("fft", 9, 12, 8192, 8192, 8192) == K["fft1p"]
    assert _device.compress_kernel("fft", 3, 12, 16384, 16384, 16384) == K["fft2p"]  # columns exceed smem
    assert _device.compress_kernel("fwht", 3, 6, 100, 100, 100) == K["fold"]         # b < 2^8
