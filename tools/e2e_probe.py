"""Break the host-to-host (e2e) cfg3 step into its parts on cuda:0."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from paper_2601_09477_b200 import _device, workloads as W  # noqa: E402

dev = torch.device("cuda")
w = W.make("cfg3", xp=torch, device=dev)
p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
a_h = w.a.cpu().pin_memory()
b_h = w.bmat.cpu().pin_memory()
est_h = torch.empty((w.n, w.n), dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream()


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} {e0.elapsed_time(e1) / reps:9.2f} ms (wall {1e3 * (time.perf_counter() - t0) / reps:9.2f})",
          flush=True)
    return out


buf = torch.empty_like(w.a)
timed("H2D 2 GiB contiguous", lambda: buf.copy_(a_h, non_blocking=True))
timed("D2H 2 GiB contiguous", lambda: est_h.copy_(buf, non_blocking=True))
cs = torch.cuda.Stream()
slab = torch.empty((w.n, 2048), dtype=torch.float64, device=dev)


def cols():
    for c0 in range(0, w.n, 2048):
        _device.copy2d(slab, a_h[:, c0:c0 + 2048], s)


timed("H2D 2 GiB as 8 column slabs (2-D)", cols)
sk = timed("compress(host A, B) streamed", lambda: P.compress(a_h, b_h, p))
timed("compress(device A, B)", lambda: P.compress(w.a, w.bmat, p))
timed("extract_all -> host est", lambda: P.extract_all(sk, w.threshold, strict=True, est_out=est_h))
est_d = torch.empty((w.n, w.n), dtype=torch.float64, device=dev)
_, pairs = timed("extract_all -> device est", lambda: P.extract_all(sk, w.threshold, strict=True, est_out=est_d))
timed("pairs D2H", lambda: pairs.to("cpu"))


def e2e_step():
    sk2 = P.compress(a_h, b_h, p)
    _, pairs2 = P.extract_all(sk2, w.threshold, strict=True, est_out=est_h)
    return pairs2


timed("e2e step (compress host + extract host)", e2e_step)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk2 = P.compress(a_h, b_h, p)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, pairs2 = P.extract_all(sk2, w.threshold, strict=True, est_out=est_h)
    t2 = time.perf_counter()
    print(f"phases: compress {1e3 * (t1 - t0):.1f} ms, extract {1e3 * (t2 - t1):.1f} ms", flush=True)
