"""Per-configuration measurement of every BASELINE config on cuda:0 (round evidence).

For each config: device time of compress (plan + kernel + inverse) and of the
fused extraction + threshold (CUDA events, median of reps, inputs resident),
the FP64 roofline fraction of compress against the measured pipe peak, and the
CPU oracle (the bit-exact port of the reference algorithm, all host threads) on
a bounded k-slice / row-slice of the same instance, extrapolated.

    python tools/config_bench.py [cfg ...]  ->  profiles/<round>_configs.{json,md}  (SMM_ROUND, default r02)
    python tools/config_bench.py --from-log LOG   (tables from a run's printed JSON lines)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_09477_b200 as P  # noqa: E402
from oracle import sketch_oracle as O  # noqa: E402
from paper_2601_09477_b200 import _device, workloads as W  # noqa: E402

ROUND = __import__("os").environ.get("SMM_ROUND", "r02")

FP64_OPS_PEAK = 18.52e12  # DADD / DFMA per second (profiles/r01_microbench.txt)
DEFAULT = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5_b12_d3_nnz512_fwht", "cfg5_b12_d5_nnz512_fft",
           "cfg5_b14_d9_nnz512_fwht", "cfg5_b14_d9_nnz512_fft", "cfg5_b16_d9_nnz512_fwht",
           "cfg5_b16_d3_nnz512_fft", "cfg5_b18_d3_nnz512_fwht", "cfg5_b18_d3_nnz512_fft",
           "cfg5_b20_d3_nnz512_fwht", "cfg5_b20_d3_nnz512_fft"]


def fp64_ops(n, b, d, transform):
    lb = b.bit_length() - 1
    if transform == "fwht":  # transforms, products, scatters, inverse, scale
        return 2 * d * n * b * lb + d * n * b + 2 * d * n * n + d * b * lb + d * b
    # packed complex FFT: (b/2) log2 b radix-2 butterflies of 8 pipe ops (twiddle product: 2 MUL +
    # 2 FMA, then 4 adds) per (t, k); FA/FB split + product + accumulate ~6 per bucket; scatters 2
    # per input; one inverse per repetition
    return d * n * (4 * b * lb + 6 * b) + 2 * d * n * n + 4 * d * b * lb


def gpu_times(w, reps=5):
    p = P.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
    est = torch.empty((w.n, w.n), dtype=torch.float64, device="cuda")
    tc, tx = [], []
    # small configurations finish six runs in a few ms, before an idle GPU has left its idle clocks
    # (cfg1 measured 0.34 ms right after an idle gap, 0.21 ms warm): run warm for >= 0.3 s first
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.3:
        P.extract_all(P.compress(w.a, w.bmat, p), w.threshold, strict=True, est_out=est)
        torch.cuda.synchronize()
    _device.kernel_timing_read(0), _device.kernel_timing_read(1)
    for i in range(reps + 1):
        if i == 1:
            _device.kernel_timing(True)  # the compress kernel's own launches (fwht2p / fft2p), warm runs only
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        sk = P.compress(w.a, w.bmat, p)
        e1.record()
        _, pairs = P.extract_all(sk, w.threshold, strict=True, est_out=est)
        e2.record()
        torch.cuda.synchronize()
        tc.append(e0.elapsed_time(e1))
        tx.append(e1.elapsed_time(e2))
    _device.kernel_timing(False)
    ktot, kn = _device.kernel_timing_read(0)
    _device.kernel_timing_read(1)
    return float(np.median(tc[1:])), float(np.median(tx[1:])), int(pairs.shape[0]), sk, ktot / max(kn, 1)


def dgemm_ms(w):
    """cuBLAS DGEMM (torch.matmul float64) of the same A, B: context only."""
    if w.n > 16384:
        return None
    c = torch.matmul(w.a, w.bmat)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        c = torch.matmul(w.a, w.bmat)
    e1.record()
    torch.cuda.synchronize()
    del c
    return e0.elapsed_time(e1) / 2


def cpu_time(w, threads, budget_s=6.0):
    words = O.draw_words(w.sketch_seed, w.d, w.b)
    n = w.n

    def run(ks, rs):
        a = w.a[:, :ks].cpu().numpy()
        bm = w.bmat[:ks].cpu().numpy()
        t0 = time.perf_counter()
        polys = O.compress(a, bm, b=w.b, d=w.d, words=words, transform=w.transform, seed=0, threads=threads)
        tk = time.perf_counter() - t0
        t0 = time.perf_counter()
        est, _, _ = O.decompress(polys, words, b=w.b, d=w.d, transform=w.transform, n1=n, n2=n, r0=0, r1=rs,
                                 want_est=True, threads=threads)
        np.argwhere(np.abs(est) > w.threshold)  # the reference's threshold (experiments.py:136-168)
        return tk, time.perf_counter() - t0

    tk, tr = run(8, 16)
    ks = int(min(n, max(8, 0.7 * budget_s / max(tk / 8, 1e-9))))
    rs = int(min(n, max(16, 0.3 * budget_s / max(tr / 16, 1e-9))))
    tk, tr = run(ks, rs)
    return (tk * n / ks + tr * n / rs) * 1e3, ks, rs


def main(names):
    threads = O.cpu_count()
    O.build()
    rows = []
    for name in names:
        w = W.make(name, xp=torch, device="cuda")
        tcomp, text, hh, sk, tkern = gpu_times(w)
        ops = fp64_ops(w.n, w.b, w.d, w.transform)
        cpu_ms, ks, rs = cpu_time(w, threads)
        gemm = dgemm_ms(w)
        row = {"config": name, "n": w.n, "b": w.b, "d": w.d, "transform": w.transform,
               "compress_ms": tcomp, "compress_kernel_ms": tkern, "extract_ms": text, "total_ms": tcomp + text,
               "heavy_hitters": hh, "fp64_ops": ops, "fp64_frac": ops / (tcomp * 1e-3) / FP64_OPS_PEAK,
               "fp64_frac_kernel": ops / (tkern * 1e-3) / FP64_OPS_PEAK, "dgemm_ms": gemm,
               "extract_write_gbs": 8 * w.n * w.n / (text * 1e-3) / 1e9,
               "cpu_oracle_ms": cpu_ms, "cpu_threads": threads, "cpu_sample": f"k {ks}/{w.n}, rows {rs}/{w.n}",
               "speedup_vs_cpu": cpu_ms / (tcomp + text)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del w, sk
        torch.cuda.empty_cache()
    write_tables(rows)


def write_tables(rows):
    out = ROOT / "profiles" / f"{ROUND}_configs.json"
    out.write_text(json.dumps(rows, indent=1))
    lines = ["| config | transform | n | b | d | compress ms (kernel) | FP64 frac (kernel) | extract ms | "
             "est. write GB/s | CPU oracle ms (threads) | speed-up | DGEMM ms (context) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        gemm = f"{r['dgemm_ms']:.1f}" if r.get("dgemm_ms") else "-"
        lines.append(f"| {r['config']} | {r['transform']} | {r['n']} | 2^{r['b'].bit_length() - 1} | {r['d']} | "
                     f"{r['compress_ms']:.2f} ({r.get('compress_kernel_ms', float('nan')):.2f}) | "
                     f"{100 * r['fp64_frac']:.1f} % ({100 * r.get('fp64_frac_kernel', float('nan')):.1f} %) | "
                     f"{r['extract_ms']:.2f} | "
                     f"{r['extract_write_gbs']:.0f} | {r['cpu_oracle_ms']:.0f} ({r['cpu_threads']}) | "
                     f"{r['speedup_vs_cpu']:.0f}x | {gemm} |")
    (ROOT / "profiles" / f"{ROUND}_configs.md").write_text(
        f"# {ROUND} per-configuration measurements (B200, one GPU)\n\n"
        "Device time with inputs resident (CUDA events, median of 5): compress through the API (B-slab\n"
        "transpose, hash plans, the compress kernel, inverse) and, in parentheses, the compress kernel's own\n"
        "launches (fwht2p / fft2p, CUDA events on the launching stream); FP64 fraction against the measured\n"
        "18.52 T ops/s pipe peak (FFT: radix-2 butterflies counted as pipe ops); CPU: the bit-exact oracle\n"
        "port of the reference algorithm on all host threads over a bounded k-slice and row-slice of the\n"
        "same instance, extrapolated (tools/config_bench.py); cuBLAS DGEMM of the same A, B as context\n"
        "(n <= 16384).\n\n" + "\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1:2] == ["--from-log"]:  # rebuild the tables from the JSON lines of a GPU-box run
        write_tables([json.loads(ln) for ln in open(sys.argv[2]) if ln.startswith("{")])
    else:
        main(sys.argv[1:] or DEFAULT)
