"""Per-step device times of the bench step (cfg3: compress + extract_all), with
and without the nvidia-smi clock sampler running, to find step-time outliers."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import workloads as W  # noqa: E402

w = W.make("cfg3", xp=torch, device="cuda")
p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
est_buf = torch.empty((w.n, w.n), dtype=torch.float64, device="cuda")


def step():
    sk = P.compress(w.a, w.bmat, p)
    P.extract_all(sk, w.threshold, strict=True, est_out=est_buf)


for _ in range(3):
    step()
torch.cuda.synchronize()
for sampler in (False, True, False, True):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    ev[0].record()
    for i in range(8):
        step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    if ctx:
        ctx.__exit__(None, None, None)
    print("sampler" if sampler else "plain  ", " ".join(f"{ev[i].elapsed_time(ev[i + 1]):7.2f}" for i in range(8)),
          flush=True)
