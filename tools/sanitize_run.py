"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every
product-path kernel family on cfg1-sized inputs — fwht2p (pair and one-k-per-lane
mappings, fold b > 2^16, accumulate mode), fft2p (plain and folded), the v1 fold
kernels (b < 2^8), the d > 63 path, hash tables, finalize, extraction + pair list
and batched queries.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import _device  # noqa: E402

rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
a = torch.as_tensor(rng.standard_normal((n, n)), device="cuda")
b = torch.as_tensor(rng.standard_normal((n, n)), device="cuda")
cases = [("fwht", 1 << 12, 3), ("fwht", 1 << 9, 5), ("fwht", 1 << 17, 3), ("fwht", 1 << 6, 3),
         ("fft", 1 << 12, 3), ("fft", 1 << 15, 3), ("fft", 1 << 6, 3), ("fwht", 1 << 8, 65)]
for tr, width, d in cases:
    p = P.SketchParams(n=n, b=width, d=d, transform=tr, seed=3)
    sk = P.compress(a, b, p)
    est, pairs = P.extract_all(sk, 2.0, strict=True)
    q = P.decompress_entries(sk, np.array([[0, 1], [n - 1, 2]]))
    print(tr, width, d, float(sk.polys_device().abs().sum()), int(pairs.shape[0]), q.shape, flush=True)
# odd k range (one-k-per-lane mapping) and accumulate mode over two calls
words = P.SketchHashes.draw(np.random.default_rng(4), 3, 1 << 12).packed_words()
acc = _device.compress_accumulate(a[:, :99], b[:99], words, 3, 12, "fwht", 0, 99, a_layout=_device.KMINOR)
_device.compress_accumulate(a[:, 99:], b[99:], words, 3, 12, "fwht", 0, n - 99, acc=acc, a_layout=_device.KMINOR,
                            accumulate=True)
# host-resident operands (streamed k-slabs) and host extraction
sk = P.compress(a.cpu().numpy(), b.cpu().numpy(), P.SketchParams(n=n, b=1 << 12, d=3, seed=5))
est_h = torch.empty((n, n), dtype=torch.float64).pin_memory()
P.extract_all(sk, 2.0, strict=True, est_out=est_h)
torch.cuda.synchronize()
print("sanitize workload done", flush=True)
