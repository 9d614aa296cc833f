"""Ad-hoc GPU parity sweep against the committed golden fixtures (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402

g = np.load(ROOT / "tests/golden/small_cases.npz")
bad = 0
for name in g["names"]:
    name = str(name)
    n1, m, n2, b, d, seed, th, isf = (int(x) for x in g[f"{name}/meta"])
    tr = "fwht" if isf else "fft"
    a, bm = g[f"{name}/a"], g[f"{name}/b"]
    p = P.SketchParams(n=m, b=b, d=d, transform=tr, seed=seed)
    try:
        sk = P.compress_rect(a, bm, p) if (n1 != m or n2 != m) else P.compress(a, bm, p)
        ref = g[f"{name}/polys"]
        err = np.abs(sk.polys - ref).max() / max(1.0, np.abs(ref).max())
        est = P.decompress_all(sk)
        eref = g[f"{name}/est"]
        eerr = np.abs(est - eref).max() / max(1.0, np.abs(eref).max())
        exact = np.array_equal(sk.polys, ref)
        ok = err < 1e-12 and eerr < 1e-12
    except Exception as exc:  # noqa: BLE001
        ok, err, eerr, exact = False, float("nan"), float("nan"), False
        print("EXC", name, exc)
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} {name:45s} polys_rel={err:.2e} est_rel={eerr:.2e} exact={exact}")
print("bad:", bad)
sys.exit(1 if bad else 0)
