"""Per-rank work of the N-GPU sharded product, measured on one GPU.

For N in {1, 2, 4, 8}, rank g of the k-sharded path (paper_2601_09477_b200.distributed)
runs: compress of its k-slab (B-slab transpose, CSR plan, fwht2p), the inverse, and
the extraction + threshold of its n/N output rows.  This times exactly that work for
the slowest rank on cuda:0 (inputs resident, CUDA events, median of reps); the one
collective (a d x b float64 allreduce) is not run here (one GPU per call) and is
listed by size.  Output: one JSON line per N, and profiles/<SMM_ROUND>_scaling_model_<cfg>.json.

    python tools/scaling_model.py [cfg3|cfg4]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import _device, workloads as W  # noqa: E402
from paper_2601_09477_b200.distributed import row_bounds, shard_bounds  # noqa: E402
from paper_2601_09477_b200.hashing import SketchHashes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = 5
w = W.make(cfg, xp=torch, device="cuda")
p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
hashes = SketchHashes.draw(np.random.default_rng(p.seed), p.d, p.b)
words = hashes.packed_words()
rows = []
for world in (1, 2, 4, 8):
    worst = None
    for rank in (0, world - 1):  # slabs are equal up to one index; time the first and the last
        k0, k1 = shard_bounds(w.n, world, rank)
        r0, r1 = row_bounds(w.n, world, rank)
        a_slab, b_slab = w.a[:, k0:k1], w.bmat[k0:k1]
        est = torch.empty((r1 - r0, w.n), dtype=torch.float64, device="cuda")

        def rank_step():
            acc = _device.compress_accumulate(a_slab, b_slab, words, p.d, p.log2b, p.transform, 0, k1 - k0,
                                              a_layout=_device.KMINOR)
            polys = _device.finalize(acc, p.d, p.log2b, p.transform)
            sk = P.ProductSketch(polys, hashes, p, w.n, w.n)
            return P.extract_all(sk, w.threshold, strict=True, r0=r0, r1=r1, est_out=est)

        out = rank_step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = rank_step()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        worst = t if worst is None else max(worst, t)
        del out, est
    acc_bytes = 8 * p.d * p.b if p.transform == "fwht" else 16 * p.d * (p.b // 2 + 1)
    row = {"config": cfg, "n_gpus": world, "rank_ms": worst, "allreduce_bytes": acc_bytes if world > 1 else 0}
    rows.append(row)
    print(json.dumps(row), flush=True)
base = rows[0]["rank_ms"]
for r in rows:
    r["speedup_vs_1"] = base / r["rank_ms"]
    r["efficiency"] = base / (r["rank_ms"] * r["n_gpus"])
out = ROOT / "profiles" / f"{__import__('os').environ.get('SMM_ROUND', 'r02')}_scaling_model_{cfg}.json"
out.write_text(json.dumps(rows, indent=1))
print(json.dumps(rows))
