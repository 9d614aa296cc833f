"""Benchmark of the sketched-product hot path on B200 (BASELINE.json metric).

Workload: BASELINE cfg3 — n = 16384 float64, FWHT variant, b = 2^16, d = 5,
+-1 operands with 256 planted heavy entries (paper_2601_09477_b200/workloads.py),
heavy-hitter threshold |est| > n/2.  One *step* is one complete sketched
product through the public API on device-resident operands:
  compress (A^T transpose, hash plans, fused fold-scatter + FWHT + product +
  accumulate, CTA-partial reduction, inverse FWHT and 1/b) followed by
  extraction of all n^2 median estimates (materialised in HBM) fused with the
  heavy-hitter threshold and the row-major pair list.
Metric: milliseconds per sketched product (lower is better).  With N ranks
(torchrun) the inner dimension is sharded (k-slab per rank), the d x b
accumulators are summed with one NCCL allreduce, and output rows are sharded:
same total work, strong scaling; the reported time is the max over ranks.

``--impl reference`` times the reference algorithm's CPU implementation (the
bit-exact C/OpenMP oracle port, oracle/, all host cores) running the FULL product
of the same workload every step (A^T copy, compress over all n inner indices,
inverse, all n^2 estimates, threshold and pair list) — no extrapolation.  When
the unmodified reference package is installed in baseline/_ref
(tools/install_reference.sh), one full run of its own Numba path (sketchmm.compress
+ decompress_all + threshold) is added as ``cpu_baseline.detail.stock_reference``.
Our arm also lists cuBLAS DGEMM (torch.matmul, float64) on the same A, B as
context (the reference's timing harness does the same, experiments.py:505-516).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sketched_product_ms_n16384_fp64"
UNIT = "ms"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "_fallback": True}


# measured on this pool's B200 by tools/microbench.cu (profiles/r01_microbench.txt):
# DADD 18.52 Tops/s = 63.7 FP64-pipe ops/clk/SM at 1965 MHz (burst, kernel timed alone)
FP64_PIPE_PEAK_TOPS = 18.52


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm
def _oracle_sample(w, k_slice: int, row_slice: int, threads: int):
    """Time the CPU oracle (reference algorithm, bit-exact port) on a bounded sample of w:
    the A^T copy and compress of a k-slice, the inverse, the estimates of a row slice and
    their threshold, each scaled to the full product (the same steps _oracle_full times)."""
    from oracle import sketch_oracle as O

    words = O.draw_words(w.sketch_seed, w.d, w.b)
    t0 = time.perf_counter()
    at = np.ascontiguousarray(w.a[:, :k_slice].T)  # rows k of A^T for the k-slice (as the reference copies A.T)
    acc = O.accumulate_fwht(at, w.bmat[:k_slice], b=w.b, d=w.d, words=words, k0=0, k1=k_slice, threads=threads)
    tk = time.perf_counter() - t0
    del at
    t0 = time.perf_counter()
    polys = O.fwht_inverse_scaled(acc)
    tf = time.perf_counter() - t0
    t0 = time.perf_counter()
    est, _, _ = O.decompress(polys, words, b=w.b, d=w.d, transform=w.transform, n1=w.n, n2=w.n, r0=0,
                             r1=row_slice, want_est=True, threads=threads)
    hh = np.argwhere(np.abs(est) > w.threshold)  # the reference's threshold (experiments.py:136-168)
    tr = time.perf_counter() - t0
    full_ms = (tk * w.n / k_slice + tf + tr * w.n / row_slice) * 1e3
    return full_ms, {"k_slice": k_slice, "row_slice": row_slice, "t_k_s": tk, "t_rows_s": tr, "t_inv_s": tf,
                     "heavy_hitters_in_rows": int(hh.shape[0])}


def _cpu_instance(cfg: str):
    from paper_2601_09477_b200 import workloads as W

    return W.make(cfg)


def _calibrate(w, threads: int, budget_s: float):
    _, info = _oracle_sample(w, 16, 64, threads)
    per_k = info["t_k_s"] / 16
    per_row = info["t_rows_s"] / 64
    k_slice = int(min(w.n, max(16, (0.7 * budget_s) / max(per_k, 1e-9))))
    row_slice = int(min(w.n, max(64, (0.3 * budget_s) / max(per_row, 1e-9))))
    return k_slice, row_slice


def _oracle_full(w, threads: int):
    """One full sketched product on the CPU oracle (the reference's algorithm, bit-exact
    port): A^T copy (sketch.py:305), compress over every inner index, inverse, all n^2
    estimates (sketch.py:375-399), then the reference's threshold — numpy over the
    estimate matrix, as experiments.py:136-168 does — giving the row-major pair list."""
    from oracle import sketch_oracle as O

    words = O.draw_words(w.sketch_seed, w.d, w.b)
    t0 = time.perf_counter()
    at = np.ascontiguousarray(w.a.T)
    acc = O.accumulate_fwht(at, w.bmat, b=w.b, d=w.d, words=words, k0=0, k1=w.n, threads=threads)
    del at
    t1 = time.perf_counter()
    polys = O.fwht_inverse_scaled(acc)
    t2 = time.perf_counter()
    est, _, _ = O.decompress(polys, words, b=w.b, d=w.d, transform=w.transform, n1=w.n, n2=w.n, want_est=True,
                             threads=threads)
    t3 = time.perf_counter()
    hh = np.argwhere(np.abs(est) > w.threshold)
    t4 = time.perf_counter()
    return (t4 - t0) * 1e3, {"compress_s": t1 - t0, "inverse_s": t2 - t1, "decompress_s": t3 - t2,
                             "threshold_s": t4 - t3, "heavy_hitters": int(hh.shape[0])}


def _stock_reference(w):
    """One full run of the unmodified reference (baseline/_ref, Numba) on the same inputs, or why not."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "sketchmm").exists():
        return {"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    sys.path.insert(0, str(ref_dir))
    try:
        import numba
        from sketchmm import sketch as RS

        threads = int(numba.config.NUMBA_NUM_THREADS)
        # JIT warm-up on a small instance of the same dtypes
        small = np.ones((64, 64))
        RS.decompress_all(RS.compress(small, small, RS.SketchParams(n=64, b=1 << 8, d=w.d, seed=1), threads=threads))
        p = RS.SketchParams(n=w.n, b=w.b, d=w.d, transform=w.transform, seed=w.sketch_seed)
        t0 = time.perf_counter()
        sk = RS.compress(w.a, w.bmat, p, threads=threads)
        t1 = time.perf_counter()
        est = RS.decompress_all(sk)
        t2 = time.perf_counter()
        hh = np.argwhere(np.abs(est) > w.threshold)
        t3 = time.perf_counter()
        return {"value_ms": (t3 - t0) * 1e3, "compress_s": t1 - t0, "decompress_all_s": t2 - t1,
                "threshold_s": t3 - t2, "heavy_hitters": int(hh.shape[0]), "threads": threads,
                "numba": numba.__version__, "note": "unmodified sketchmm from baseline/_ref, one run after a "
                                                    "small JIT warm-up; informational"}
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:300]}
    finally:
        sys.path.remove(str(ref_dir))


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import sketch_oracle as O

    O.build()
    threads = O.cpu_count()
    w = _cpu_instance(args.config)
    times = []
    info = None
    # warm-up steps: a bounded sample of the same work (the C port has no JIT; this warms the
    # OpenMP pool and the caches), so the driver's W warm-ups do not cost W full products
    for step in range(args.warmup):
        ms, _ = _oracle_sample(w, min(w.n, 512), min(w.n, 512), threads)
        print(f"reference warm-up {step}: sample (k 512, rows 512)", file=sys.stderr, flush=True)
    for step in range(args.steps):
        ms, info = _oracle_full(w, threads)
        print(f"reference step {step}: {ms:.0f} ms {info}", file=sys.stderr, flush=True)
        times.append(ms)
    value = float(np.median(times))
    sample = (f"oracle C/OpenMP port (bit-exact vs reference Numba kernels) on {threads} host threads: the full "
              f"n={w.n} product every step (A^T copy, compress over all inner indices, inverse, all n^2 "
              f"estimates, threshold + pair list); median of {args.steps} steps")
    stock = _stock_reference(w) if not args.no_stock_reference else {"unavailable": "--no-stock-reference"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE cfg3 construction)",
            "config": _config(args, w.n, w.b, w.d),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "detail": {"last_step": info, "stock_reference": stock}},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(args, n, b, d):
    return {"workload": f"BASELINE {args.config}: n={n} fp64 FWHT b={b} d={d}, +-1 operands with 256 planted "
                        f"entries, heavy-hitter threshold |est|>n/2; compress + inverse + full n^2 extraction + threshold",
            "n": n, "b": b, "d": d, "transform": "fwht", "parallelism": f"k-shard x{args.gpus} + 1 allreduce",
            "l2": "operands (2 x 2 GiB) exceed the 126 MB L2; no flush needed between steps"}


TRAFFIC_FILE = ROOT / "profiles" / "compress_dram_bytes.json"


def _kernel_source_sha() -> str:
    import hashlib

    h = hashlib.sha256()
    for f in ("fwht2p.cu", "twopass.cuh", "plan.cuh", "common.cuh"):
        h.update((ROOT / "paper_2601_09477_b200" / "csrc" / f).read_bytes())
    return h.hexdigest()[:16]


def _traffic():
    """DRAM bytes per fwht2p launch from the committed ncu --set full capture, used only
    if that capture was taken of the kernel source built here (sha match); else null."""
    try:
        rec = json.loads(TRAFFIC_FILE.read_text())
    except Exception:  # noqa: BLE001
        return None, "no ncu capture committed"
    if rec.get("kernel_source_sha") != _kernel_source_sha():
        return None, f"stale: {TRAFFIC_FILE.name} was captured from another fwht2p source"
    return rec.get("dram_bytes_per_launch"), f"{TRAFFIC_FILE.name} ({rec.get('report')})"


L2_WRITE_TBS = 7.57  # L2-resident store bandwidth (tools/microbench.cu)
L2_READ_TBS = 17.5   # L2-resident read bandwidth
GATHERS_PER_S = 294.4e9  # random 8-byte gathers (1.00 per clk per SM)


def _l2_view(kl: int, b: int, d: int, t_ms: float) -> dict:
    lb = b.bit_length() - 1
    bs = 1 << min(lb, 16)              # two-pass slice size (fold above 2^16)
    units = -(-kl // 32) * d * (b // bs)
    y = 2 * units * bs * 32 * 8        # both operands, one 32-wide k-tile per unit
    floor_ms = (y / (L2_WRITE_TBS * 1e12) + y / (L2_READ_TBS * 1e12)) * 1e3
    return {"y_bytes_written": y, "y_bytes_read": y, "floor_ms": floor_ms, "frac": floor_ms / t_ms,
            "peaks_tbs": {"write": L2_WRITE_TBS, "read": L2_READ_TBS}}


# ----------------------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2601_09477_b200 as P
    from paper_2601_09477_b200 import _device, _lib, workloads as W
    from paper_2601_09477_b200.distributed import compress_sharded, row_bounds, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N-rank path on a one-GPU box only (never a measurement):
    # SMM_BENCH_SAME_DEVICE=1 puts every rank on cuda:0, SMM_BENCH_BACKEND=gloo avoids
    # NCCL's one-rank-per-device rule
    if os.environ.get("SMM_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SMM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator set-up (transport, NVLS) on stderr: the JSON line stays alone on stdout
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lib = _lib.load()

    w = W.make(args.config, xp=torch, device=dev)
    n, b, d = w.n, w.b, w.d
    params = P.SketchParams(n=n, b=b, d=d, transform=w.transform, seed=w.sketch_seed)
    k0, k1 = shard_bounds(n, world, rank)
    r0, r1 = row_bounds(n, world, rank)
    # this rank's device-resident inputs: the k-slab of A (a column view, no copy) and of B (rows)
    a_slab = w.a[:, k0:k1]
    b_slab = w.bmat[k0:k1]
    est_buf = torch.empty((r1 - r0, n), dtype=torch.float64, device=dev)

    def step():
        if world == 1:
            sk = P.compress(w.a, w.bmat, params)
        else:
            sk = compress_sharded(a_slab, b_slab, params, n_rows=n, n_cols=n, a_layout=_device.KMINOR)
        est, pairs = P.extract_all(sk, w.threshold, strict=True, r0=r0, r1=r1, est_out=est_buf)
        return sk, est, pairs

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up holds the previous step's outputs while the next step runs, exactly as the timed
    # loop does, so the caching allocator reaches its steady state (no cudaMalloc while timed)
    sk = est = pairs = None
    for _ in range(args.warmup):
        sk, est, pairs = step()
    barrier()
    launches0 = lib.smm_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # live per-launch timing of the dominant kernels: CUDA events recorded by the library
    # around each fwht2p / extract launch on its stream, inside the timed steps
    _device.kernel_timing_read(0), _device.kernel_timing_read(1)  # drop anything recorded earlier
    _device.kernel_timing(True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record()
        evs = []
        for _ in range(args.steps):
            sk, est, pairs = step()
            evs.append(torch.cuda.Event(enable_timing=True))
            evs[-1].record()
        ev1.record()
        barrier()
    _device.kernel_timing(False)
    comp_total, comp_n = _device.kernel_timing_read(0)
    ext_total, ext_n = _device.kernel_timing_read(1)
    per_step = [ev0.elapsed_time(evs[0])] + [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
    print("per-step ms: " + " ".join(f"{x:.2f}" for x in per_step), file=sys.stderr, flush=True)
    launches = lib.smm_kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    hh_local = int(pairs.shape[0])

    # ---- the dominant kernel's average launch duration over the timed steps (for the roofline)
    kl = k1 - k0
    t_comp = comp_total / max(comp_n, 1)
    t_extract = ext_total / max(ext_n, 1)
    logb = params.log2b
    # algorithmic FP64-pipe ops of one accumulate launch: 2 forward transforms per (k, t),
    # one product-accumulate FMA per bucket, one signed scatter-add per input element
    ops = 2 * d * kl * b * logb + d * kl * b + 2 * d * kl * n
    achieved = ops / (t_comp * 1e-3) / 1e12
    hbm_bytes = 16 * n * kl + 8 * d * b
    roofline = {"bound": "fp64", "kernel": "fwht2p_kernel; average of its launches inside the timed "
                                            "steps, CUDA events recorded on the launching stream (smm_kernel_timing)",
                "launches_timed": comp_n, "achieved": achieved,
                "peak": FP64_PIPE_PEAK_TOPS, "unit": "Tops/s", "frac": achieved / FP64_PIPE_PEAK_TOPS,
                "traffic": None, "algorithmic_ops": ops, "kernel_ms": t_comp,
                "peak_source": "measured DADD pipe rate, tools/microbench.cu (profiles/r01_microbench.txt); "
                               "MEASURED_PEAKS.json holds no FP64 figure",
                "hbm": {"algorithmic_bytes": hbm_bytes, "achieved_gbs": hbm_bytes / (t_comp * 1e-3) / 1e9,
                        "peak_gbs": _peaks().get("hbm_gbs"),
                        "frac": hbm_bytes / (t_comp * 1e-3) / 1e9 / _peaks().get("hbm_gbs", 6650.0)},
                "extract": {"ms": t_extract, "launches_timed": ext_n, "algorithmic_bytes": 8 * (r1 - r0) * n,
                            "achieved_gbs": 8 * (r1 - r0) * n / (t_extract * 1e-3) / 1e9,
                            # d random 8-byte gathers per estimate, one L1 line lookup each (1/clk/SM,
                            # profiles/r01_microbench.txt "gather8"): the binding resource
                            "gathers": d * (r1 - r0) * n,
                            "gather_floor_ms": d * (r1 - r0) * n / GATHERS_PER_S * 1e3,
                            "frac_of_gather_floor": d * (r1 - r0) * n / GATHERS_PER_S * 1e3 / t_extract},
                # the pass-1 -> pass-2 intermediate Y crosses L2 once per element and operand:
                # written at <= 7.57 TB/s and read at <= 17.5 TB/s (measured, profiles/r01_microbench.txt)
                "l2": _l2_view(kl, b, d, t_comp)}
    roofline["traffic"], roofline["traffic_source"] = _traffic()

    # ---- e2e through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        a_host = a_slab.contiguous().cpu().pin_memory()
        b_host = b_slab.contiguous().cpu().pin_memory()
        est_host = torch.empty((r1 - r0, n), dtype=torch.float64).pin_memory()
        torch.cuda.empty_cache()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def e2e_step():
            if world == 1:
                sk2 = P.compress(a_host, b_host, params)
            else:
                sk2 = compress_sharded(a_host, b_host, params,
                                       n_rows=n, n_cols=n, a_layout=_device.KMINOR)
            # host destination: row blocks are copied out while the next block extracts
            _, pairs2 = P.extract_all(sk2, w.threshold, strict=True, r0=r0, r1=r1, est_out=est_host)
            return pairs2  # pinned host tensor, complete on return

        for _ in range(2):  # two warm-ups: the pinned pair buffers of consecutive steps alternate
            hp = e2e_step()
        barrier()
        e0.record()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            hp = e2e_step()
        e1.record()
        barrier()
        e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": float(e2e_ms.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(a_host.numel() * 8 + b_host.numel() * 8),
               "d2h_bytes_per_step": int(est_host.numel() * 8 + hp.numel() * 8),
               "path": "paper_2601_09477_b200.compress(pinned host tensors; k-slabs uploaded while earlier slabs "
                       "compute) + extract_all(est_out=pinned host rows; row blocks copied out while the next "
                       "extracts; heavy-hitter pairs returned in pinned host memory)"}

    # ---- context only: cuBLAS DGEMM of the same A, B (the dense product the sketch replaces)
    dgemm = None
    if not args.no_dgemm:
        try:
            c = torch.matmul(a_slab, b_slab)
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            reps = 3
            for _ in range(reps):
                c = torch.matmul(a_slab, b_slab)
            g1.record()
            torch.cuda.synchronize()
            gms = g0.elapsed_time(g1) / reps
            del c
            dgemm = {"ms": gms, "tflops": 2.0 * n * (k1 - k0) * n / (gms * 1e-3) / 1e12,
                     "what": "torch.matmul float64 (cuBLAS DGEMM) of this rank's A[:, k-slab] @ B[k-slab, :], "
                             "n x n output; context only (reference experiments.py:505-516 times the dense "
                             "product beside the sketch)"}
        except RuntimeError as exc:  # e.g. out of memory
            dgemm = {"unavailable": str(exc)[:200]}

    # ---- CPU baseline (rank 0, N=1): bounded oracle sample on the host cores
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import sketch_oracle as O

        O.build()
        threads = O.cpu_count()
        wc = _cpu_instance(args.config)
        k_slice, row_slice = _calibrate(wc, threads, args.cpu_budget)
        full_ms, info = _oracle_sample(wc, k_slice, row_slice, threads)
        cpu_baseline = {"value": full_ms, "unit": UNIT, "cores": threads, "kind": "port",
                        "sample": f"oracle C/OpenMP port on {threads} host threads: compress k-slice {k_slice}/{n}, "
                                  f"decompress+threshold rows {row_slice}/{n}, extrapolated to the full product",
                        "detail": info}

    if rank == 0:
        line = {"metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE cfg3 construction, seeded)",
                "config": _config(args, n, b, d), "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk.summary(),
                "breakdown_ms": {"compress_accumulate": t_comp, "extract_all": t_extract},
                "context_dgemm": dgemm,
                "heavy_hitters_rank0": hh_local}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--no-dgemm", action="store_true", help="skip the cuBLAS DGEMM context timing")
    ap.add_argument("--no-stock-reference", action="store_true",
                    help="--impl reference: skip the one run of the unmodified reference (baseline/_ref)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
