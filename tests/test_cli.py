"""The CLI multiply workflow (reference cli.py:133-199) and its matrix files
(reference matio.py): formats pinned against files the reference wrote
(tests/golden/matrix_ref.*, tools/make_golden.py matrix)."""
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

import paper_2601_09477_b200 as P
from paper_2601_09477_b200 import matio
from paper_2601_09477_b200.cli import main
from paper_2601_09477_b200.errors import FormatError

GOLD = Path(__file__).parent / "golden"


def test_matrix_files_match_the_reference_bytes(tmp_path):
    m = np.load(GOLD / "matrix_ref.npy")
    assert matio.matrix_to_bytes(m) == (GOLD / "matrix_ref.dmat").read_bytes()
    assert np.array_equal(matio.load_matrix(GOLD / "matrix_ref.dmat"), m)
    back = matio.load_matrix(GOLD / "matrix_ref.csv")
    assert np.array_equal(back, m)  # %.17g round-trips float64
    matio.save_matrix(tmp_path / "m.csv", m)
    assert (tmp_path / "m.csv").read_bytes() == (GOLD / "matrix_ref.csv").read_bytes()


def test_matrix_format_errors():
    raw = (GOLD / "matrix_ref.dmat").read_bytes()
    with pytest.raises(FormatError):
        matio.matrix_from_bytes(raw[:10])
    with pytest.raises(FormatError):
        matio.matrix_from_bytes(b"XMAT" + raw[4:])
    with pytest.raises(FormatError):
        matio.matrix_from_bytes(raw[:-8])


def test_cli_usage_errors_exit_2(tmp_path):
    a = tmp_path / "a.dmat"
    matio.save_matrix(a, np.eye(8))
    r = CliRunner().invoke(main, ["multiply", str(a), str(a), "-o", str(tmp_path / "o.dmat")])
    assert r.exit_code == 2 and "either --cd with --cb" in r.output
    r = CliRunner().invoke(main, ["multiply", str(a), str(a), "-o", str(tmp_path / "o"), "--cd", "1"])
    assert r.exit_code == 2
    r = CliRunner().invoke(main, ["multiply", str(a), str(a), "-o", str(tmp_path / "o"), "-b", "6", "-d", "3"])
    assert r.exit_code == 2 and "power of two" in r.output  # InvalidParameterError -> usage error
    bad = tmp_path / "bad.dmat"
    bad.write_bytes(b"nope")
    r = CliRunner().invoke(main, ["multiply", str(bad), str(a), "-o", str(tmp_path / "o"), "-b", "16", "-d", "3"])
    assert r.exit_code == 1  # FormatError -> runtime failure


@pytest.mark.gpu
def test_cli_multiply_writes_estimates_and_sketch(tmp_path):
    rng = np.random.default_rng(4)
    n = 256
    a = rng.integers(-3, 4, size=(n, n)).astype(np.float64)
    b = rng.integers(-3, 4, size=(n, n)).astype(np.float64)
    matio.save_matrix(tmp_path / "a.dmat", a)
    matio.save_matrix(tmp_path / "b.csv", b)
    for transform in ("fwht", "fft"):
        out, skp = tmp_path / f"est_{transform}.dmat", tmp_path / f"{transform}.skch"
        r = CliRunner().invoke(main, ["--seed", "9", "--transform", transform, "multiply", str(tmp_path / "a.dmat"),
                                      str(tmp_path / "b.csv"), "-o", str(out), "-b", "2048", "-d", "5",
                                      "--save-sketch", str(skp)])
        assert r.exit_code == 0, r.output
        p = P.SketchParams(n=n, b=2048, d=5, transform=transform, seed=9)
        sk = P.compress(a, b, p)
        assert np.array_equal(matio.load_matrix(out), P.decompress_all(sk))
        assert P.load_sketch(skp) == sk


def test_cli_global_options_max_mem_and_format(tmp_path):
    """--max-mem applies the reference's budget check (cli.py:85-92) before any device
    work: an over-budget run exits 1; --format is accepted (reference global option)."""
    a = tmp_path / "a.dmat"
    matio.save_matrix(a, np.eye(64))
    args = ["multiply", str(a), str(a), "-o", str(tmp_path / "o.dmat"), "-b", "4096", "-d", "5"]
    r = CliRunner().invoke(main, ["--max-mem", "1K"] + args)
    assert r.exit_code == 1 and "exceeds --max-mem" in r.output
    r = CliRunner().invoke(main, ["--max-mem", "lots"] + args)
    assert r.exit_code == 2
    need = int(1.25 * P.estimate_workspace_bytes(64, 4096, 5, "fwht", 1))
    assert need > 1024
    r = CliRunner().invoke(main, ["--format", "xml"] + args)
    assert r.exit_code == 2
    from paper_2601_09477_b200.cli import _parse_bytes

    assert _parse_bytes("4G") == 4 << 30 and _parse_bytes("1.5k") == 1536 and _parse_bytes("10") == 10
