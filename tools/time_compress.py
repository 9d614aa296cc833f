"""Device time of P.compress on named workloads (median of reps), cuda:0."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import workloads as W  # noqa: E402

reps = int(__import__("os").environ.get("REPS", "5"))
for name in sys.argv[1:]:
    w = W.make(name, xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.compress(w.a, w.bmat, p)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[1:])
    print(f"{name:28s} compress median {ts[len(ts) // 2]:8.3f} ms  min {ts[0]:8.3f}  max {ts[-1]:8.3f}", flush=True)
    if __import__("os").environ.get("ALL"):
        print("   ", " ".join(f"{x:.2f}" for x in ts))
