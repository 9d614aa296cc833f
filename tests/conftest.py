import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def small_cases():
    g = np.load(GOLDEN / "small_cases.npz")
    cases = []
    for name in g["names"]:
        name = str(name)
        n1, m, n2, b, d, seed, th, isf = (int(x) for x in g[f"{name}/meta"])
        cases.append({
            "name": name, "n1": n1, "m": m, "n2": n2, "b": b, "d": d, "seed": seed, "threads": th,
            "transform": "fwht" if isf else "fft", "a": g[f"{name}/a"], "bm": g[f"{name}/b"],
            "polys": g[f"{name}/polys"], "est": g[f"{name}/est"], "words": g[f"{name}/words"],
        })
    return cases


@pytest.fixture(scope="session")
def hash_golden():
    return json.loads((GOLDEN / "hash_golden.json").read_text())


@pytest.fixture(scope="session")
def draws_golden():
    return json.loads((GOLDEN / "draws.json").read_text())["draws"]


@pytest.fixture(scope="session")
def transforms_golden():
    return json.loads((GOLDEN / "transforms.json").read_text())


def cfg_golden(name: str):
    p = GOLDEN / f"{name}.npz"
    return np.load(p) if p.exists() else None
