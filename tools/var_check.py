"""sha256 of the sketches of a few workloads under the loaded library (SMM_LIB): variants
of a kernel must reproduce the product library's bits (dev tool for tools/ab.sh runs)."""
import hashlib
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import workloads as W  # noqa: E402

for name in sys.argv[1:] or ["cfg3", "cfg1", "cfg5_b14_d5_nnz8192_fwht", "cfg5_b18_d3_nnz512_fwht"]:
    w = W.make(name, xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    sk = P.compress(w.a, w.bmat, p)
    torch.cuda.synchronize()
    print(f"{name:28s} polys sha {hashlib.sha256(sk.polys.tobytes()).hexdigest()[:16]}", flush=True)
