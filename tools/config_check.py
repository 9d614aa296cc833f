"""Dev tool: GPU sketch of BASELINE configs vs the reference goldens + timings."""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import workloads as W  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
for name in names:
    gp = ROOT / "tests/golden" / f"{name}.npz"
    g = np.load(gp)
    t0 = time.time()
    w = W.make(name, xp=torch, device="cuda")
    torch.cuda.synchronize()
    tgen = time.time() - t0
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        sk = P.compress(w.a, w.bmat, p)
        torch.cuda.synchronize()
        tc = time.time() - t0
        t0 = time.time()
        est = P.decompress_rows(sk)
        torch.cuda.synchronize()
        td = time.time() - t0
    polys = sk.polys
    sha = hashlib.sha256(np.ascontiguousarray(polys).tobytes()).hexdigest()
    gsha = bytes(g["polys_sha256"]).decode()
    samp = np.take_along_axis(polys, g["polys_sample_idx"], axis=1)
    perr = np.abs(samp - g["polys_sample"]).max()
    scale = max(1.0, np.abs(g["polys_sample"]).max())
    if "polys" in g:
        perr = np.abs(polys - g["polys"]).max()
    ij = g["est_sample_ij"]
    e = est[torch.as_tensor(ij[:, 0], device="cuda"), torch.as_tensor(ij[:, 1], device="cuda")].cpu().numpy()
    eerr = np.abs(e - g["est_sample"]).max()
    hh = P.heavy_hitters(sk, w.threshold, True)
    hsha = hashlib.sha256(np.ascontiguousarray(hh.astype(np.int64)).tobytes()).hexdigest()
    print(f"{name}: gen {tgen:.2f}s compress {tc*1e3:.2f} ms extract {td*1e3:.2f} ms | polys sha match={sha == gsha} "
          f"max|dpolys|={perr:.3e} (scale {scale:.3e}) max|dest|={eerr:.3e} hh={hh.shape[0]} vs {int(g['hh_count'][0])} "
          f"hh_sha_match={hsha == bytes(g['hh_sha256']).decode()}", flush=True)
    del w, sk, est
    torch.cuda.empty_cache()
