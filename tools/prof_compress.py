"""Profiling driver: one warm cfg3 compress (accumulate) + one extraction on cuda:0.

    ncu --set full -k regex:fwht_fold -c 1 python tools/prof_compress.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import _device, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = W.make(cfg, xp=torch, device="cuda")
p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
words = P.SketchHashes.draw(__import__("numpy").random.default_rng(p.seed), p.d, p.b).packed_words()
bt = w.bmat.T.contiguous()
for _ in range(reps):
    acc = _device.compress_accumulate(w.a, bt, words, p.d, p.log2b, p.transform, 0, w.n,
                                      a_layout=_device.KMINOR, b_layout=_device.KMINOR)
    polys = _device.finalize(acc, p.d, p.log2b, p.transform)
    sk = P.ProductSketch(polys, P.SketchHashes.from_words(words, p.d, p.b), p, w.n, w.n)
    est, pairs = P.extract_all(sk, w.threshold, strict=True)
torch.cuda.synchronize()
print("done", float(polys.abs().sum()), int(pairs.shape[0]))
