#!/usr/bin/env python
"""LOVE / KISS-GP hot-path benchmark (contract: one JSON line on rank 0).

A step = one pass of the whole hot path of SURVEY.md §8(a) over one batch of synthetic
input: love_build_cache (interpolation + sort, k Lanczos steps with full
reorthogonalisation, streamed Cholesky / Rc / mean cache, + the sampling root for config 5)
followed by predict_var on the t test points (+ s joint draws for config 5).  Workload at
N=1: BASELINE.json configs[1] (config 2: n=1e6, m=1e5, k=100, t=1e6, fp32 with fp64
reductions).

N>1 (one rank per GPU; `--gpus N` without torchrun re-launches itself under
torch.distributed.run on 127.0.0.1):
  --scaling weak   : every rank holds its own full-size n-point shard (seeded by rank) of one
                     global training set and its own t test points (per-GPU work fixed);
  --scaling strong : ONE global draw of the config (seed 0) is split with shard_bounds: rank r
                     owns a contiguous 1/N of the n training points and of the t test points
                     (total work fixed; BASELINE config 4: "training points sharded over 8 GPUs").
  Default: strong for config 4, weak otherwise.  The per-step exchange is NCCL over NVLink
  inside the library (all-reduces of u, alpha, the reorthogonalisation dots, beta^2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl love|reference] [--config 2]
                  [--scaling auto|weak|strong]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "predictive variances/sec + LOVE cache-build ms at n,m,k; % of HBM roofline"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP32_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_fp32_peak.json")
FALLBACK_HBM_GBS = 6650.0      # /opt/skills/guides/B200_PROFILING.md fallback
REF_BUDGET_S = 240.0           # wall-clock budget of the reference arm's K + W steps


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="love", choices=["love", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanczos", default="full", choices=["full", "partial"],
                    help="partial: opt-in partial reorthogonalisation (SURVEY 8(f) NEXT #1); the default "
                         "hot path reorthogonalises fully every step")
    return ap.parse_args(argv)


def scaling_mode(p, requested: str) -> str:
    if requested != "auto":
        return requested
    return "strong" if p.name.startswith("cfg4") else "weak"


def self_launch(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-run this script under torch.distributed.run with
    N ranks on 127.0.0.1.  Returns the launcher's exit code, or None when no launch is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def fp32_peak():
    """FP32 FMA peak (TFLOP/s) of the sampling roofline: the FFMA2 microbenchmark
    tools/ubench/fma_peak.cu measured on this pool's B200 (profiles/r02_fp32_peak.json), else
    the unit-count figure 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz = 74.4 TFLOP/s."""
    try:
        with open(FP32_PEAK_FILE) as f:
            d = json.load(f)
        return float(d["ffma2_tflops"]), "measured (profiles/r02_fp32_peak.json, FFMA2 microbenchmark)"
    except Exception:
        return 148 * 128 * 2 * 1.965e9 / 1e12, "derived (148 SMs x 128 lanes x 2 FLOP x 1965 MHz)"


def reorth_bytes(n_local: int, k: int, vsize: int, passes: int = 1) -> dict:
    """Algorithmic bytes of the reorthogonalisation kernels over one build:
    step j (0-based, j < k-1) with c = j+1 stored columns:
      dots   : c*n*s_v (Q~ columns) + n*s_v (r)
      update : c*n*s_v (Q~ columns) + n*s_v (r) + n*s_v (new column written)"""
    dots = upd = 0
    for j in range(k - 1):
        ccols = j + 1
        dots += passes * (ccols * n_local * vsize + n_local * vsize)
        upd += passes * (ccols * n_local * vsize + 2 * n_local * vsize)
    return {"dots": dots, "update": upd}


def build_bytes(p, n_local: int, k: int | None = None) -> int:
    """Algorithmic bytes of one cache build, SURVEY.md §8(d):
    B_step(j) = n (2 r_d + 5 s_v) + 2 n j s_v + 4 m s_v  (j = 1..k), B_build = sum_j B_step(j)
    + 2 m k s_v, with s_v the vector element size and r_d = 8d (fp32) / 12d (fp64) bytes of a
    point's record.  ONE CGS pass, as the survey grades the build ("graded against the one-pass
    model"); fp64 runs CGS2, whose second pass the dominant-kernel roofline counts instead."""
    k = p.k if k is None else k
    fp64 = p.precision == "fp64" or p.cache_fp64
    sv, rd = (8, 12 * p.d) if fp64 else (4, 8 * p.d)
    tot = 0
    for j in range(1, k + 1):
        tot += n_local * (2 * rd + 5 * sv) + 2 * n_local * j * sv + 4 * p.m_total * sv
    return tot + 2 * p.m_total * k * sv


def query_bytes(p, k_pad: int, t: int | None = None, occupied_cells: int | None = None):
    """Algorithmic bytes of one variance query and the model used.
    d <= 2 (per-cell variance blocks, SURVEY §8(f) #3b): the fp64 query point, the packed fp64
    block of its cell (4^d (4^d + 1) / 2 values) and the result.
    d = 3 (cell-sorted queries, SURVEY §8(f) #3a): per query the fp64 point, its sort key and
    permutation entry (written and read back: 4 x 4 B) and the result; per OCCUPIED cell the 64
    stencil rows of Rc staged once (64 k_pad s_R) -- amortised over the t queries when t and the
    occupied-cell count are given, else SURVEY §8(d)'s gathered-row upper bound 4^d k s_R."""
    sv = 8 if p.precision == "fp64" else 4
    sr = 8 if (p.precision == "fp64" or p.cache_fp64) else 4
    if p.kind == "additive":
        return 4 * p.d * k_pad * sr + 8 * p.d + sv, "gathered rows of the 4d block stencil (Eq. 16)"
    if p.d <= 2:
        nb = 4 ** p.d
        return 8 * p.d + 8 * nb * (nb + 1) // 2 + sv, "cell-block (x*, fp64 block of its cell, result)"
    if t and occupied_cells:
        per = 8 * p.d + 16 + sv + 64 * k_pad * sr * occupied_cells / t
        return per, (f"cell-sorted: x*, key/perm, result per query + 64 Rc rows per occupied cell "
                     f"({occupied_cells} cells for {t} queries)")
    return 4 ** p.d * k_pad * sr + 8 * p.d + sv, "gathered rows (SURVEY 8(d) B_query)"


def occupied_cells(p, Xs: np.ndarray) -> int:
    """Number of distinct interpolation cells floor((x - lo) / h) among the test points (the
    cells whose Rc rows the d = 3 sorted query kernel stages); bookkeeping of the byte model."""
    h = np.array(p.h)
    lo = np.array(p.lo)
    cell = np.floor((Xs - lo) / h).astype(np.int64)
    key = np.zeros(len(Xs), dtype=np.int64)
    for d in range(p.d):
        key = key * p.m[d] + cell[:, d]
    return int(np.unique(key).size)


def sample_flops(t: int, ks: int, s: int, d: int) -> dict:
    """FLOPs of one love_sample call: the draw product G zeta (t x k' by k' x s,
    2 t k' s) plus the gather G = W*^T S (2 4^d t k')."""
    return {"gemm": 2 * t * ks * s, "gather": 2 * (4 ** d) * t * ks}


class ClockSampler:
    """SM clock and throttle-reason sampling DURING the timed region (the recipe's clocks
    line).  NVML is polled from a thread every ~2 ms (nvidia-smi -lms cannot resolve a
    timed region of tens of ms); `nvidia-smi` is the fallback when NVML is unavailable."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.idx = gpu_index
        self.period = period_s
        self.sm, self.reasons, self.smax = [], set(), None
        self.stop_ev = threading.Event()
        self.thread = None
        self.err = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        except Exception as e:                       # no NVML: no clocks record
            self.err = f"nvml unavailable: {e}"
            return
        self.N, self.h = N, h
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        t0 = time.time()
        while not self.sm and time.time() - t0 < 2.0:   # first sample before the region starts
            time.sleep(0.001)

    def _run(self):
        N, h = self.N, self.h
        while not self.stop_ev.is_set():
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                mask = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                for nm, attr in self.REASONS:
                    if mask & getattr(N, attr, 0):
                        self.reasons.add(nm)
            except Exception as e:
                self.err = str(e)
                break
            time.sleep(self.period)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"], "samples": 0}
        self.stop_ev.set()
        self.thread.join(timeout=2)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 2 ms polling"}


# ----------------------------------------------------------------------------- workload
def shard_inputs(p, rank: int, world: int, scaling: str):
    """This rank's inputs.  weak: its own full-size draw (seed p.seed + rank); strong: rank r's
    contiguous shard_bounds slice of the ONE global draw (seed p.seed) of X, y and X*."""
    from paper_1803_06058_b200.dist import shard_bounds
    from synth import make_inputs
    from synth.inputs import Inputs
    if scaling == "weak" or world == 1:
        return make_inputs(p, seed=p.seed + rank)
    g = make_inputs(p, seed=p.seed)
    lo, hi = shard_bounds(p.n, rank, world)
    tlo, thi = shard_bounds(p.t, rank, world)
    return Inputs(g.X[lo:hi], g.y[lo:hi], g.Xs[tlo:thi])


def config_record(p, world: int, scaling: str) -> dict:
    """The `config` object of BOTH arms' JSON lines (identical keys and values)."""
    per_gpu = scaling == "weak" or world == 1
    return {"workload": p.name, "n": p.n * (world if per_gpu else 1), "m": p.m_total, "k": p.k,
            "t": p.t * (world if per_gpu else 1), "d": p.d, "precision": p.precision,
            "cache": "fp64" if (p.precision == "fp64" or p.cache_fp64) else "fp32",
            "k_sample": p.k_sample, "s": p.s,
            "l2": "flushed (256 MB write) between timed steps",
            "parallelism": f"dp{world} ({scaling} scaling: training + test points sharded, "
                           "NCCL all-reduce per Lanczos step)"}


# ----------------------------------------------------------------------------- oracle arm
def run_oracle_step(p, inp, t_sample):
    """One step of the fp64 CPU oracle: paper-literal build (+ the sampling root for config 5)
    + variance queries (+ s draws) on t_sample test points.  Returns (build_s, query_s)."""
    import oracle as O
    from synth import make_zeta
    t0 = time.perf_counter()
    if p.kind == "additive":
        model = O.build_model_additive(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, [p.outputscale] * p.d,
                                       p.sigma2)
    else:
        model = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
    cache = O.love_precompute(model, p.k)
    sc = O.sampling_cache(model, cache, p.k_sample) if p.k_sample else None
    t1 = time.perf_counter()
    Xs = inp.Xs[:t_sample]
    O.predict_var(model, cache, Xs)
    if sc is not None:
        O.draw_samples(model, cache, sc, Xs, make_zeta(sc.lanczos.k_eff, p.s))
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(p, inp, t_sample=50_000):
    """The oracle as it stands, on this host's cores, full build + a bounded query sample
    (at most the t test points); the query time is scaled to the full t (queries are
    independent and O(k) each)."""
    t_sample = min(t_sample, len(inp.Xs))
    b, q = run_oracle_step(p, inp, t_sample)
    scale = len(inp.Xs) / t_sample
    step = b + q * scale
    what = "predict_var" + (f" + {p.s} draws" if p.k_sample else "")
    return {"value": len(inp.Xs) / step, "unit": "variances/s", "cores": oracle_threads(), "kind": "oracle",
            "sample": f"full {p.name} build (n={len(inp.X)}, m={p.m_total}, k={p.k}"
                      + (f", sampling root k'={p.k_sample}" if p.k_sample else "") + f") + {what} on {t_sample} "
                      f"of {len(inp.Xs)} test points" + (f", query time scaled x{scale:.0f}" if scale > 1 else ""),
            "build_s": round(b, 3), "query_s_sample": round(q, 3)}


def reference_arm(args, p):
    """The oracle timed as run: every step is a full oracle build plus queries on a bounded
    prefix of the test points, sized so the K + W steps fit REF_BUDGET_S; `value` is the
    variances that step computed over its measured time (no extrapolation)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import make_inputs
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    scaling = scaling_mode(p, args.scaling)
    inp = make_inputs(p)
    b0, q0 = run_oracle_step(p, inp, min(p.t, 20_000))        # calibration, untimed
    per_point = q0 / min(p.t, 20_000)
    per_step = REF_BUDGET_S / max(1, args.steps + args.warmup)
    t_sample = int(min(p.t, max(min(p.t, 20_000), (per_step - b0) / max(per_point, 1e-12))))
    for _ in range(args.warmup):
        run_oracle_step(p, inp, t_sample)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run_oracle_step(p, inp, t_sample)
        times.append(time.perf_counter() - t0)
    step = float(np.mean(times))
    value = t_sample / step
    what = "predict_var" + (f" + {p.s} draws" if p.k_sample else "")
    sample = (f"each step as run: full {p.name} oracle build (n={p.n}, m={p.m_total}, k={p.k}"
              + (f", sampling root k'={p.k_sample}" if p.k_sample else "")
              + f") + {what} on the first {t_sample} of {p.t} test points; value = {t_sample} variances / "
                "measured step time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "variances/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_record(p, world, scaling),
        "cpu_baseline": {"kind": "oracle", "cores": oracle_threads(), "sample": sample, "value": value,
                         "unit": "variances/s"},
        "e2e": {"value": value, "unit": "variances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- LOVE arm
def main():
    args = parse()
    rc = self_launch(args) if args.impl == "love" else None
    if rc is not None:
        raise SystemExit(rc)
    from synth import get_config
    p = get_config(args.config)
    if args.impl == "reference":
        reference_arm(args, p)
        return

    import torch
    import torch.distributed as dist
    from paper_1803_06058_b200 import LoveCache, launch_count, nccl_unique_id
    from paper_1803_06058_b200 import _abi
    from paper_1803_06058_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    scaling = scaling_mode(p, args.scaling)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl_id = D.nccl_id_for_group(make_id=nccl_unique_id)

    inp = shard_inputs(p, rank, world, scaling)
    n_loc, t_loc = len(inp.X), len(inp.Xs)
    X = torch.from_numpy(inp.X).to(dev)
    y = torch.from_numpy(inp.y).to(dev)
    Xs = torch.from_numpy(inp.Xs).to(dev)
    kw = dict(m=p.m, lo=p.lo, h=p.h, lengthscale=p.lengthscale, outputscale=p.outputscale, sigma2=p.sigma2,
              k=p.k, precision=p.precision, rank=rank, world=world, nccl_id=nccl_id, k_sample=p.k_sample,
              cache_fp64=True if p.cache_fp64 else "auto")
    lib = _abi.load()
    if p.kind == "additive":                      # Eq. 16 block forms (NEXT #2): no sampling cache
        kw.pop("k_sample")
    if args.lanczos == "partial":
        kw["lanczos_mode"] = "partial"

    def build(Xd, yd):
        if p.kind == "additive":
            return LoveCache.build_additive(Xd, yd, **kw)
        return LoveCache.build(Xd, yd, **kw)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    lib.love_profile_enable(0)

    def step(Xd, yd, Xsd):
        c = build(Xd, yd)
        var = c.predict_var(Xsd)
        if p.k_sample:
            c.sample(Xsd, p.s, seed=0)
        c.free()
        return var

    # end to end: X, y (pinned host) go through LoveCache.build, which uploads them on the
    # current stream; the test points are uploaded on a side stream (ordered after the step's
    # start event, so the copy is inside the timed span) while the build runs; the variances
    # (and draws) come back into pinned host buffers.  Every copy is inside the step.
    side = torch.cuda.Stream(device=dev)

    def step_e2e(Xh, yh, Xsh, outs, start_ev):
        side.wait_event(start_ev)
        with torch.cuda.stream(side):
            Xsd = Xsh.to(dev, non_blocking=True)
            up = torch.cuda.Event()
            up.record(side)
        c = build(Xh, yh)
        torch.cuda.current_stream().wait_event(up)
        Xsd.record_stream(torch.cuda.current_stream())
        var = c.predict_var(Xsd)
        outs[0].copy_(var, non_blocking=True)
        if p.k_sample:
            outs[1].copy_(c.sample(Xsd, p.s, seed=0).t(), non_blocking=True)   # (s, t) storage
        c.free()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(X, y, Xs)
    barrier()

    # ---------------- timed region: K steps, device events, L2 flushed between steps.  The
    # production path runs (each build replays its Lanczos step as a CUDA graph).
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = launch_count()
    total_ms = 0.0
    build_ms, query_ms, sample_ms = [], [], []
    k_pad, n_reorth, k_eff, ks_eff, cache_prec = 0, 0, 0, 0, 0
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        e0.record(stream)
        c = build(X, y)
        e1.record(stream)
        c.predict_var(Xs)
        e2.record(stream)
        if p.k_sample:
            c.sample(Xs, p.s, seed=0)
        e3.record(stream)
        e3.synchronize()
        total_ms += e0.elapsed_time(e3)
        build_ms.append(e0.elapsed_time(e1))
        query_ms.append(e1.elapsed_time(e2))
        sample_ms.append(e2.elapsed_time(e3))
        inf = c.info()
        k_pad, n_reorth, k_eff = inf["k_pad"], inf["n_reorth_steps"], inf["k_eff"]
        ks_eff, cache_prec = inf["k_sample_eff"], inf["cache_precision"]
        c.free()
    barrier()
    launches = launch_count() - launches0
    clk = clocks.stop()
    ms_per_step = D.max_over_ranks(total_ms / args.steps, dev)
    t_total = D.sum_over_ranks(float(t_loc), dev)
    value = t_total / (ms_per_step / 1e3)

    # ---------------- phase timing: the same steps with CUDA events around every phase's
    # kernels on the launching stream (eager launches: events cannot sit inside the graph)
    import ctypes
    nprof = max(1, min(2, args.steps))
    lib.love_profile_read(None, None, 1)
    lib.love_profile_enable(1)
    prof_step_ms = 0.0
    for _ in range(nprof):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c = build(X, y)
        c.predict_var(Xs)
        if p.k_sample:
            c.sample(Xs, p.s, seed=0)
        e1.record(stream)
        e1.synchronize()
        prof_step_ms += e0.elapsed_time(e1)
        c.free()
    lib.love_profile_enable(0)
    ms_arr = (ctypes.c_double * len(_abi.PROF_NAMES))()
    calls_arr = (ctypes.c_int64 * len(_abi.PROF_NAMES))()
    lib.love_profile_read(ms_arr, calls_arr, 1)
    prof_ms = {nm: ms_arr[i] / nprof for i, nm in enumerate(_abi.PROF_NAMES)}
    prof_step_ms /= nprof

    # ---------------- roofline of the dominant kernels (full reorthogonalisation)
    peak, peak_src = hbm_peak()
    vs = 8 if cache_prec == _abi.LOVE_FP64 else 4
    rb = reorth_bytes(n_loc, k_eff, vs, passes=2 if vs == 8 else 1)
    reorth_ms = prof_ms["reorth_dots"] + prof_ms["reorth_update"]
    achieved = (rb["dots"] + rb["update"]) / (reorth_ms / 1e3) / 1e9 if reorth_ms > 0 else None
    traffic, traffic_info = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tr = json.load(open(tfile)).get(p.name)
            if tr and world == 1:
                traffic = tr["bytes"]
                traffic_info = {"launches": tr["launches"], "algorithmic_bytes": tr["algorithmic_bytes"],
                                "ratio": tr["bytes"] / tr["algorithmic_bytes"], "source": "profiles/traffic.json"}
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": "reorth_dots + reorth_update (full reorthogonalisation, "
                                          "classical Gram-Schmidt, Q read twice per step)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_launches": traffic_info,
                "peak_source": peak_src,
                "algorithmic_bytes_per_build": rb["dots"] + rb["update"],
                "kernel_ms_per_build": reorth_ms,
                "share_of_step": reorth_ms / prof_step_ms if prof_step_ms else None,
                "timing": "CUDA events around the phase's launches on the launching stream, "
                          f"{nprof} eager step(s) run right after the timed region"}

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(inp.X).pin_memory()
        yh = torch.from_numpy(inp.y).pin_memory()
        Xsh = torch.from_numpy(inp.Xs).pin_memory()
        odt = torch.float64 if p.precision == "fp64" else torch.float32
        outs = [torch.empty(t_loc, dtype=odt, pin_memory=True)]
        if p.k_sample:
            outs.append(torch.empty((p.s, t_loc), dtype=odt, pin_memory=True))
        a0 = torch.cuda.Event()
        a0.record(stream)
        step_e2e(Xh, yh, Xsh, outs, a0)             # warm the host-buffer path (allocator, pinned copies)
        barrier()
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step_e2e(Xh, yh, Xsh, outs, a)
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        te = D.max_over_ranks(tot / args.steps, dev)
        e2e = {"value": t_total / (te / 1e3), "unit": "variances/s",
               "h2d_bytes_per_step": int(inp.X.nbytes + inp.y.nbytes + inp.Xs.nbytes),
               "d2h_bytes_per_step": int(sum(o.numel() * o.element_size() for o in outs)), "ms_per_step": te,
               "note": "per rank (each rank copies its own shard)" if world > 1 else None}

    # whole-build and query roofline fractions under SURVEY §8(d)'s byte model
    bb = build_bytes(p, n_loc, k_eff)
    b_ach = bb / (float(np.mean(build_ms)) / 1e3) / 1e9
    build_rf = {"bound": "hbm", "algorithmic_bytes": bb, "achieved": b_ach, "peak": peak, "unit": "GB/s",
                "frac": b_ach / peak,
                "model": f"SURVEY 8(d) B_build at k_eff = {k_eff} (one CGS pass = 2 reads of Q_j per step)"}
    # achieved = bytes / the query kernels' own time (CUDA events around their launches in the
    # profiled steps); the step's query_ms also holds the host gap of the Python call
    occ = occupied_cells(p, inp.Xs) if (p.kind != "additive" and p.d == 3) else None
    bq, qmodel = query_bytes(p, k_pad, t_loc, occ)
    qb = bq * t_loc
    qk_ms = prof_ms.get("query", 0.0) or float(np.mean(query_ms))
    q_ach = qb / (qk_ms / 1e3) / 1e9
    query_rf = {"bound": "hbm", "model": qmodel, "algorithmic_bytes": qb,
                "achieved": q_ach, "peak": peak, "unit": "GB/s", "frac": q_ach / peak,
                "bytes_per_query": bq, "kernel_ms": qk_ms,
                "timing": "CUDA events around the query launches (profiled steps)"}
    if p.kind != "additive" and p.d == 3 and occ:
        # the cell-sorted kernel reads its rows from shared memory: its bound is the FP32 FMA
        # pipe -- per query and k value the separable contraction sum_a w0 sum_b w1 sum_c w2 R
        # takes 64 + 16 + 4 FMAs (2 FLOP each)
        fpk, fsrc = fp32_peak()
        qfl = 2.0 * 84 * k_eff * t_loc
        q_tf = qfl / (qk_ms / 1e3) / 1e12
        query_rf["alu"] = {"bound": "alu", "flop": qfl, "achieved": q_tf, "peak": fpk, "unit": "TFLOP/s",
                           "frac": q_tf / fpk, "peak_source": fsrc,
                           "model": "t * k_eff * (64 + 16 + 4) FMA of the per-query separable contraction"}
    if p.kind != "additive" and p.d <= 2:
        # the cell-block table (m blocks) is L2-resident: the DRAM floor is each query's x* and
        # result plus the table once, far below the gathered bytes
        nb = 4 ** p.d
        ub = t_loc * (8 * p.d + (8 if p.precision == "fp64" else 4)) + p.m_total * 8 * nb * (nb + 1) // 2
        query_rf["unique_dram_bytes"] = ub
        query_rf["unique_dram_frac"] = ub / (qk_ms / 1e3) / 1e9 / peak
        query_rf["note"] = ("frac counts the block bytes each query gathers (mostly L2 hits: the table is "
                            f"{p.m_total * 8 * nb * (nb + 1) // 2 / 1e6:.0f} MB); unique_dram_frac the DRAM floor")
    sampling = None
    if p.k_sample:
        smean = float(np.mean(sample_ms))
        fl = sample_flops(t_loc, ks_eff, p.s, p.d)
        fpk, fsrc = fp32_peak()
        gemm_ms = prof_ms.get("sample_gemm", 0.0)
        g_ach = fl["gemm"] / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
        sampling = {"s": p.s, "t": t_loc, "k_sample_eff": ks_eff, "sample_ms": smean,
                    "joint_samples_per_s": world * p.s / (smean / 1e3),
                    "sample_values_per_s": world * p.s * t_loc / (smean / 1e3),
                    "note": "draws only (Philox zeta + W*^T S zeta + mean); the sampling cache is in build_ms",
                    "roofline": {"bound": "alu", "kernel": "sample_gemm2 (F = mu 1^T + G zeta, FFMA2)",
                                 "flop": fl["gemm"], "achieved": g_ach, "peak": fpk, "unit": "TFLOP/s",
                                 "frac": g_ach / fpk if g_ach else None, "peak_source": fsrc,
                                 "kernel_ms": gemm_ms, "whole_call_ms": prof_ms.get("sample", 0.0),
                                 "whole_call_flop": fl["gemm"] + fl["gather"]}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(p, inp)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "variances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if p.precision == "fp32" else "f64", "data": "synthetic",
            "config": config_record(p, world, scaling),
            "n_local": n_loc, "t_local": t_loc, "k_eff": k_eff,
            "cache_precision": "fp64" if cache_prec == _abi.LOVE_FP64 else "fp32",
            "build_ms": float(np.mean(build_ms)),
            "query_ms": float(np.mean(query_ms)),
            "query_variances_per_s": t_loc / (float(np.mean(query_ms)) / 1e3),
            "build_roofline": build_rf, "query_roofline": query_rf,
            "sampling": sampling,
            "lanczos": {"reorthogonalisation": args.lanczos, "steps_reorthogonalised": n_reorth},
            "phase_ms_per_step": {k: round(v, 4) for k, v in prof_ms.items() if v > 0},
            "profiled_step_ms": prof_step_ms,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
