"""Per-kernel device time of P.compress (and optionally extraction) on named workloads,
from torch.profiler (CUPTI) — a launch list without nsys.

    python tools/kernel_list.py cfg5_b12_d3_nnz8192_fwht [cfg1 ...]
"""
import os
import sys
from collections import defaultdict
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import workloads as W  # noqa: E402

reps = int(os.environ.get("REPS", "3"))
for name in sys.argv[1:]:
    w = W.make(name, xp=torch, device="cuda")
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    for _ in range(2):
        P.compress(w.a, w.bmat, p)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            P.compress(w.a, w.bmat, p)
        torch.cuda.synchronize()
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            tot[ev.name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            cnt[ev.name] += 1
    all_us = sum(tot.values()) / reps
    print(f"== {name}: {all_us / 1000:.3f} ms of device time per compress")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v / reps / 1000:8.3f} ms  x{cnt[k] // reps:<3d} {k[:110]}")
