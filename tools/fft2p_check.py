"""fft2p against the CPU oracle on random operands (dev tool): b = 2^8 .. 2^14, partial k tiles."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import sketch_oracle as O  # noqa: E402
from paper_2601_09477_b200 import _device  # noqa: E402

bad = 0
for log2b, n1, m, n2, d in ((8, 300, 70, 200, 3), (10, 500, 100, 400, 5), (12, 700, 33, 650, 3), (14, 1000, 64, 900, 3),
                            (9, 64, 40, 80, 1), (11, 2000, 96, 1500, 3), (13, 300, 50, 300, 5),
                            (15, 500, 40, 450, 3), (16, 700, 33, 650, 3), (17, 300, 64, 300, 1), (18, 400, 32, 350, 3)):
    rng = np.random.default_rng(log2b)
    a = rng.standard_normal((n1, m))
    bm = rng.standard_normal((m, n2))
    words = O.draw_words(log2b + 100, d, 1 << log2b)
    acc = _device.compress_accumulate(torch.from_numpy(a).cuda(), torch.from_numpy(bm).cuda(), words, d, log2b, "fft",
                                      0, m, a_layout=_device.KMINOR, b_layout=_device.KMAJOR)
    polys = _device.finalize(acc, d, log2b, "fft").cpu().numpy()
    ref = O.compress(a, bm, b=1 << log2b, d=d, words=words, transform="fft", seed=0, threads=8)
    err = np.abs(polys - ref).max() / max(1e-300, np.abs(ref).max())
    ok = err < 1e-12
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} b=2^{log2b} n1={n1} m={m} n2={n2} d={d} rel={err:.3e}", flush=True)
print("bad:", bad)
