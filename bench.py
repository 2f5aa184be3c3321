#!/usr/bin/env python
"""Benchmark: rows/sec sketched (fp32, ell given) on 1..8 B200, % of roofline, cov-err.

Workload (BASELINE.json config 4, the largest single-GPU configuration and the
one north_star's >=60% roofline / >=75% scaling targets are read on):
    noisy low-rank stream n = 8,388,608 rows, d = 1024, k = 64, zeta = 10 (32 GiB fp32),
    ell = 128, Fast FD (2*ell buffer), P_total = 2368 shard streams (16 x 148; 296 per GPU at 8 GPUs),
    rows split evenly across the N GPUs (strong scaling; the shard DAG depends on
    P_total only, so every N computes the same sketch), per-GPU sketches
    all-gathered (NCCL) and tree-merged.
A step = fd_reset + fd_append_rows(all local rows) + fd_sketch (+ all_gather +
fd_merge for N > 1), with A already resident in HBM (32 GiB >> 126 MB L2, so
every step streams A from HBM; no flush needed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2|c1] [--variant fast_fd] [--no-e2e] [--no-cpu]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rows/sec sketched (fp32, ell given) at 1/2/4/8 B200 + % roofline; cov err"
WORKLOADS = {
    # name: (fdgen config, ell, default variant, P_total) -- one per BASELINE.json config.
    # Per-row variants default to P_total = 1, the paper-exact single stream (reading C10);
    # the batched configs use the shard counts of the cached oracle parity runs.
    "c1": ("c1", 16, "fd", 1),
    "c2": ("c2", 100, "fd", 1),
    "c3": ("c3", 100, "fast_fd", 296),
    "c4": ("c4", 128, "fast_fd", 2368),
    "c5": ("c5", 32, "fd", 1),
}
GEN = {
    "c1": "noisy low-rank n=2000 d=64 k=8 zeta=10",
    "c2": "noisy low-rank n=10000 d=500 k=50 zeta=10",
    "c3": "image-like n=60000 d=3072 (rank-100 signal, [0,255] pixels / 255)",
    "c4": "noisy low-rank n=8388608 d=1024 k=64 zeta=10",
    "c5": "drifting subspaces n=200000 d=256 (20 blocks of 8-dim subspaces, fixed e every 100th row)",
}


def peaks():
    p = {"hbm_gbs": 6551.4, "bf16_tflops": 1687.5, "bf16_tflops_sustained": 1390.6, "sm_max_mhz": 1965.0,
         "source": "fallback"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        with open(f) as fh:
            p.update(json.load(fh))
        p["source"] = "measured (MEASURED_PEAKS.json)"
    # our own microbenchmarks (tools/micro/peaks.cu) for the pipes MEASURED_PEAKS.json lacks
    g = os.path.join(ROOT, "profiles", "round2_peaks_microbench.json")
    if os.path.exists(g):
        with open(g) as fh:
            m = json.load(fh)
        p.update({k: m[k] for k in ("ffma_tflops", "dfma_tflops", "tf32_tcgen05_tflops", "i8_tcgen05_tops",
                                    "i8_tcgen05_n64_tops") if k in m})
        p["micro_source"] = "measured (profiles/round2_peaks_microbench.json, tools/micro/peaks.cu)"
    return p


def retained_and_t(variant, ell, alpha):
    """(R, t): rows kept per ReduceRank and the delta index (1-based). ell-1, ell for
    every variant but the paper-literal Fast alpha-FD (C25)."""
    import math
    if variant != "fast_alpha_fd_paper":
        return ell - 1, ell
    h = max(1, math.ceil(alpha * ell / 2.0 - 1e-9))
    m = max(1, int(alpha * ell + 0.5))
    t = ell - h
    return max(ell - m, t - 1), t


def algorithmic_work(ell, d, N, R=None, t=None):
    """Algorithmic work of one ReduceRank:
    gram  = [2(ell^2-1) + (ell+1)(ell+2)] d flops (cross + new blocks; the retained
            block is diag(sigma'^2))
    recon = 4 ell (ell-1) d flops           (Wt (ell-1 x 2ell) . Bf (2ell x d))
    trd   = (4/3) N^3 flops                 (Householder tridiagonalisation)
    bt    = 2 N^2 (ell-1) flops             (back-transform of ell-1 eigenvectors)
    eig   = bisection K g iters N 5 + inverse iteration 3 J 13 N   (Sturm counts of the top K = ell
            eigenvalues, g points each per multisection iteration; 3 fp64 LDL^T solves per
            retained vector; latency-bound)
    ingest= 2 (ell+1) d 4 bytes             (read the rows, write the buffer)"""
    import math
    R = ell - 1 if R is None else R          # rows kept (diag(sigma'^2) block of the next Gram)
    t = ell if t is None else t
    nw = N - R                               # new rows per ReduceRank
    K = min(max(t, R), N)
    J = min(R, N)
    kp = 1 << max(0, (K - 1).bit_length())
    lean = 32 < N <= 256 and R <= 128
    g = max(1, min(32, (256 if lean else 512) // kp))
    iters = math.ceil(27.0 / math.log2(g + 1))
    return {
        "gram": (2 * R * nw + nw * (nw + 1)) * d,
        "recon": 2 * R * N * d,
        "trd": (4.0 / 3.0) * N ** 3,
        "bt": 2.0 * N * N * R,
        "eig": K * g * iters * N * 5.0 + 3.0 * J * 13.0 * N,
    }


def fp32_simt_peak_tflops(mhz, pk=None):
    # measured FFMA throughput (tools/micro/peaks.cu) if present, else
    # 148 SMs x 128 FP32 lanes x 2 flops (FFMA) x clock
    if pk and "ffma_tflops" in pk:
        return pk["ffma_tflops"]
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def tf32x3_peak_tflops(pk):
    # measured tcgen05 kind::tf32 throughput / 3 (3xTF32) if present, else bf16 / 2 / 3
    if "tf32_tcgen05_tflops" in pk:
        return pk["tf32_tcgen05_tflops"] / 3.0
    return pk["bf16_tflops"] / 2.0 / 3.0


# the int8 reconstruct (fd_recon_i8.cu) forms each fp32-accurate product from 9 int8
# digit products (3 W digits x 4 Bf digits, weights >= 2^16)
RECON_I8_PRODUCTS = 9


def i8_recon_peak_tflops(pk):
    # measured tcgen05 kind::i8 throughput / 9 (fp32-equivalent flops), else bf16 x 2 / 9
    return pk.get("i8_tcgen05_tops", 2.0 * pk["bf16_tflops"]) / RECON_I8_PRODUCTS


def fp64_peak_tflops(pk):
    # measured DFMA throughput if present, else 148 SMs x 64 FP64 lanes x 2 x clock
    return pk.get("dfma_tflops", 148 * 64 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return out
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        out.update(sm_mhz=statistics.median(loaded) if loaded else None, sm_max_mhz=max(mx) if mx else None,
                   reasons=reasons, samples=len(rows))
        return out


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and the --impl reference arm)
# ---------------------------------------------------------------------------
def oracle_sample(wl, rows_per_shard=None, nshards=None, variant=None, alpha=0.2, ell_override=None,
                  shards_override=None):
    """Time the oracle (as it stands) on a bounded sample of the workload: `nshards`
    shard streams of the bench DAG (one thread each, all host cores)."""
    import numpy as np  # noqa: F401
    import concurrent.futures as cf
    import fdgen
    import oracle
    cfgname, ell, v0, P = WORKLOADS[wl]
    ell = ell_override or ell
    P = shards_override or P
    variant = variant or v0
    w = fdgen.config(cfgname)
    if w.kind == fdgen.KIND_IMAGE:
        w.xminmax = fdgen.host_minmax(w)
    cores = os.cpu_count() or 1
    if P == 1:
        # one dependent stream: the oracle (one thread) on a prefix of it
        nr = min(w.n, rows_per_shard or 4000)
        A = fdgen.host_rows(w, 0, nr)
        t0 = time.perf_counter()
        oracle.sketch(A, ell, variant, alpha=alpha, nthreads=1)
        dt = time.perf_counter() - t0
        return {"value": nr / dt, "unit": "rows/s", "cores": 1, "kind": "oracle",
                "sample": f"first {nr} rows of the single {wl} stream (P_total = 1), fp64 oracle, one thread, "
                          f"{dt:.1f} s"}
    nshards = nshards or min(cores, P)
    q, r = divmod(w.n, P)
    picks = [int(s * P / nshards) for s in range(nshards)]
    jobs = []
    for s in picks:
        start = s * q + min(s, r)
        ln = q + (1 if s < r else 0)
        if rows_per_shard:
            ln = min(ln, rows_per_shard)
        jobs.append((start, ln))
    rows = [fdgen.host_rows(w, a, b) for a, b in jobs]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(nshards) as ex:
        list(ex.map(lambda A: oracle.sketch(A, ell, variant, alpha=alpha, nthreads=1), rows))
    dt = time.perf_counter() - t0
    nrows = sum(b for _, b in jobs)
    return {"value": nrows / dt, "unit": "rows/s", "cores": min(cores, nshards), "kind": "oracle",
            "sample": f"{nshards} of the {P} shard streams of {wl} ({nrows} rows, "
                      f"{'first ' + str(rows_per_shard) + ' rows of ' if rows_per_shard else ''}each shard), "
                      f"fp64 oracle, one thread per shard, {dt:.1f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = args.workload
    cfgname, ell, variant, P = WORKLOADS[wl]
    variant = args.variant or variant
    ell = args.ell or ell
    P = args.shards or P
    rows_per_shard = sample_rows(wl, P)
    times = []
    res = None
    for i in range(args.warmup + args.steps):
        res = oracle_sample(wl, rows_per_shard=rows_per_shard, variant=variant, alpha=args.alpha,
                            ell_override=ell, shards_override=P)
        if i >= args.warmup:
            times.append(res)
    vals = [t["value"] for t in times]
    value = statistics.median(vals) if vals else 0.0
    ms = [float(t["sample"].split(", ")[-1].split(" s")[0]) * 1e3 for t in times]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(ms) if ms else None,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, variant, P, world, args.alpha, ell),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": res["cores"], "kind": "oracle",
                         "sample": res["sample"]},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sample_rows(wl, P):
    """Rows per shard of the oracle's timed sample (about 10-30 s of one core per shard)."""
    if wl == "c4":
        return 2064          # 256 + 14*129 rows: 15 ReduceRanks per shard
    if P == 1:
        return {"c1": 2000, "c2": 1500, "c5": 20000}.get(wl, 4000)
    return None


def config_dict(wl, variant, P, world, alpha=None, ell=None):
    cfgname, ell0, _, _ = WORKLOADS[wl]
    ell = ell or ell0
    import fdgen
    w = fdgen.config(cfgname)
    va = f"{variant} alpha={alpha}" if (alpha is not None and "alpha" in variant) else variant
    l2 = ("inputs larger than L2 (A is streamed from HBM every step)" if w.n * w.d * 4 > 126e6 else
          "A fits in L2 (126 MB); per-row steps are latency-bound, not memory-bound")
    out = {"workload": f"{wl}: {GEN[wl]} fp32, ell={ell}, {va}, P_total={P}",
           "n": w.n, "d": w.d, "ell": ell, "variant": variant, "n_shards_total": P,
           "parallelism": f"rows dp{world}", "l2": l2}
    if alpha is not None and "alpha" in variant:
        out["alpha"] = alpha
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import fdgen
    import paper_1501_06561_b200 as fd
    from paper_1501_06561_b200.dist import gather_and_merge, local_range

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    cfgname, ell, variant, P = WORKLOADS[wl]
    variant = args.variant or variant
    ell = args.ell or ell
    P = args.shards or P
    if P % world:
        raise SystemExit(f"P_total={P} not divisible by world={world}")
    w = fdgen.config(cfgname)
    r0, r1 = local_range(w.n, rank, world, P)
    nloc = r1 - r0
    gen = fdgen.DeviceGenerator(w, device=dev)
    A = torch.empty((nloc, w.d), dtype=torch.float32, device=dev)
    gen.fill(A, r0)
    torch.cuda.synchronize()
    sk = fd.Sketcher(w.d, ell, variant, alpha=args.alpha, n_shards=P // world, device=dev)

    def step():
        sk.reset()
        sk.append(A)
        B, _ = sk.sketch(stats=False)
        if world > 1:
            B, _ = gather_and_merge(B, {"frob_sq": 0, "delta_total": 0, "removed_mass": 0, "n_shrinks": 0,
                                        "rows_seen": 0}, lambda S: sk.merge(S), None)
        return B

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    sk.profile(True)
    sk.profile_read()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        B = step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    kern = sk.profile_read()
    sk.profile(False)
    clk = clocks.stop()
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = w.n / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (live CUDA-event times of this run) ----
    pk = peaks()
    N = 2 * ell if (fd.is_batched(variant) and variant != "fast_alpha_fd_paper") else ell
    R_, t_ = retained_and_t(variant, ell, args.alpha)
    work = algorithmic_work(ell, w.d, N, R_, t_)
    sk.reset()
    sk.append(A)
    Bst, st = sk.sketch(stats=True)
    shrinks_per_step = st["n_shrinks"]
    simt_peak = fp32_simt_peak_tflops(pk.get("sm_max_mhz", 1965.0), pk)
    tf32x3 = tf32x3_peak_tflops(pk)
    # the reconstruct runs on tcgen05 kind::i8 unless FD_SIMT_RECON / FD_SIMT_GEMM (or N > 256)
    recon_tc = ((not (os.environ.get("FD_SIMT_RECON") or os.environ.get("FD_SIMT_GEMM"))) and 224 <= N <= 256
                and 112 <= R_ <= 128)   # fd_recon_i8.cu recon_i8_supported
    dom = max(kern, key=lambda k: kern[k][0])
    dom_ms = kern[dom][0] / args.steps
    perrow = dom == "perrow"
    if perrow:
        # per-row chain: f_row = 2 ell^2 d + 2 ell d flops per row (reconstruct +
        # dots), in fp64 on the FP64 pipe; latency-bound by design (n - ell + 1 dependent steps)
        flops_step = (2.0 * ell * ell * w.d + 2.0 * ell * w.d) * nloc
        roof = {"bound": "alu", "achieved": flops_step / (dom_ms / 1e3) / 1e12, "peak": fp64_peak_tflops(pk),
                "unit": "TFLOP/s"}
    elif dom == "ingest":
        bytes_step = 2.0 * nloc * w.d * 4
        roof = {"bound": "hbm", "achieved": bytes_step / (dom_ms / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s"}
    elif dom == "gram":
        flops_step = work["gram"] * shrinks_per_step
        roof = {"bound": "tensor", "achieved": flops_step / (dom_ms / 1e3) / 1e12, "peak": tf32x3,
                "unit": "TFLOP/s"}
    elif dom == "recon" and recon_tc:
        flops_step = work["recon"] * shrinks_per_step
        roof = {"bound": "tensor", "achieved": flops_step / (dom_ms / 1e3) / 1e12, "peak": i8_recon_peak_tflops(pk),
                "unit": "TFLOP/s"}
    else:
        flops_step = work[dom] * shrinks_per_step
        roof = {"bound": "alu", "achieved": flops_step / (dom_ms / 1e3) / 1e12, "peak": simt_peak, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = f"{dom}_kernel"
    roof["kernel_share_of_step"] = kern[dom][0] / ms_total
    roof["per_kernel_ms_per_step"] = {k: v[0] / args.steps for k, v in kern.items()}
    roof["launches_per_step"] = {k: v[1] / args.steps for k, v in kern.items()}
    roof["problems_per_step"] = shrinks_per_step
    micro = pk.get("micro_source")
    roof["peak_source"] = {
        "alu": (f"FP64 DFMA, {micro}" if perrow else
                (f"FP32 FFMA, {micro}" if micro else
                 f"FP32 SIMT: 148 SM x 128 lanes x 2 flop x {pk.get('sm_max_mhz', 1965.0):.0f} MHz (derived)")),
        "tensor": ((f"tcgen05 kind::i8 / {RECON_I8_PRODUCTS} (digit products per fp32-equivalent product), {micro}"
                    if dom == "recon" else f"tcgen05 kind::tf32 / 3 (3xTF32), {micro}") if micro else
                   f"3xTF32 = (bf16_tflops {pk['bf16_tflops']} / 2) / 3, {pk['source']}"),
        "hbm": f"hbm_gbs {pk['source']}"}[roof["bound"]]
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    roof["traffic"] = None
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            trj = json.load(f)
            # the captured launch names of the step kernels (tcgen05 Gram, pipelined reconstruct)
            alias = {"gram_kernel": "gram_tc_kernel",
                     "recon_kernel": "recon_i8_kernel" if recon_tc else "recon_pipe2_kernel"}
            tr = trj.get(roof["kernel"]) or trj.get(alias.get(roof["kernel"], ""))
        if tr:
            # bytes per problem from the committed capture x problems per launch of this run
            roof["traffic"] = tr["bytes_per_problem"] * shrinks_per_step / max(kern[dom][1], 1) * args.steps
            roof["traffic_source"] = tr["source"]
    # north_star roofline: slower of HBM (4d bytes/row) and the Gram + reconstruct flops
    # on the pipes this build uses (Gram: tcgen05 3xTF32; reconstruct: tcgen05 int8 digit
    # products, or FP32 SIMT where the int8 kernel does not apply)
    n_rows = w.n / world
    hbm_s = n_rows * 4 * w.d / (pk["hbm_gbs"] * 1e9)
    if perrow:
        t_roof = max(hbm_s, flops_step / (fp64_peak_tflops(pk) * 1e12))
        roof["north_star"] = {
            "R_roof_rows_per_s_per_gpu": n_rows / t_roof, "t_roof_ms": t_roof * 1e3,
            "pipes": "per-row fp64 (f_row = 2 ell^2 d + 2 ell d on the FP64 pipe, all SMs)", "hbm_ms": hbm_s * 1e3,
            "frac": (value / world) / (n_rows / t_roof),
            "note": f"{P} dependent stream(s): at most {P} x C of 148 SMs busy; latency-bound by design"}
    else:
        gram_s = work["gram"] * shrinks_per_step / (tf32x3 * 1e12)
        recon_peak = i8_recon_peak_tflops(pk) if recon_tc else simt_peak
        recon_s = work["recon"] * shrinks_per_step / (recon_peak * 1e12)
        t_roof = max(hbm_s, gram_s + recon_s)
        roof["north_star"] = {
            "R_roof_rows_per_s_per_gpu": n_rows / t_roof, "t_roof_ms": t_roof * 1e3,
            "pipes": "Gram tcgen05 3xTF32, reconstruct " + (
                f"tcgen05 int8 ({RECON_I8_PRODUCTS} digit products)" if recon_tc else "FP32 SIMT"),
            "hbm_ms": hbm_s * 1e3,
            "frac": (value / world) / (n_rows / t_roof)}
        eig_flops = (work["trd"] + work["bt"]) * shrinks_per_step
        roof["eigensolver_inclusive"] = {
            "t_roof_ms": (t_roof + eig_flops / (simt_peak * 1e12)) * 1e3,
            "frac": (ms_step / 1e3) and ((t_roof + eig_flops / (simt_peak * 1e12)) / (ms_step / 1e3))}

    gpu_launches = int(sum(v[1] for v in kern.values()))

    # ---- cov err of the final sketch (GPU evaluator, outside the timed region) ----
    from paper_1501_06561_b200.dist import dist_cov_err
    torch.cuda.synchronize()
    t_ev = time.perf_counter()
    ce = dist_cov_err(A, B, proj_k=10)
    evaluator_ms = (time.perf_counter() - t_ev) * 1e3

    # ---- e2e: host buffers through the public API, H2D + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty((nloc, w.d), dtype=torch.float32, pin_memory=True)
        Ah.copy_(A)
        del A
        torch.cuda.empty_cache()
        sk2 = sk

        def e2e_step():
            sk2.reset()
            sk2.append(Ah)              # public API: host tensor -> device copy -> fd_append_rows
            Bq, _ = sk2.sketch(stats=False)
            if world > 1:
                Bq, _ = gather_and_merge(Bq, {"frob_sq": 0, "delta_total": 0, "removed_mass": 0, "n_shrinks": 0,
                                              "rows_seen": 0}, lambda S: sk2.merge(S), None)
            return Bq.cpu()             # D2H of the result

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ks = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(ks):
            e2e_step()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        sec = float(el.item()) / ks
        e2e = {"value": w.n / sec, "unit": "rows/s", "h2d_bytes_per_step": int(w.n * w.d * 4),
               "d2h_bytes_per_step": int(ell * w.d * 4 * world), "steps": ks,
               "note": "wall clock over host-pinned input -> H2D -> sketch -> D2H of B"}

    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("f64 (per-row state and arithmetic)" if fd.is_batched(variant) is False and variant in PERROW
                  else "f32 (Gram: 3xTF32 tensor cores, fp32-accurate)"),
        "data": "synthetic (seeded fdgen, generated on device)",
        "config": config_dict(wl, variant, P, world, args.alpha, ell),
        "roofline": roof,
        "gpu_launches": gpu_launches,
        "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"]},
        "cov_err": ce["err"], "cov_err_lmin": ce["lmin"], "proj_err_k10": ce.get("proj_err"),
        "evaluator_ms": evaluator_ms,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = oracle_sample(wl, rows_per_shard=sample_rows(wl, P), variant=variant,
                                             alpha=args.alpha, ell_override=ell, shards_override=P)
    if rank == 0:
        print(json.dumps(line), flush=True)
    sk.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# Hashing / OSNAP arm: --variant osnap | hashing
# ---------------------------------------------------------------------------
HASH_S = {"osnap": 4, "hashing": 1}
PERROW = ("fd", "alpha_fd", "isvd", "ssd", "cfd")


def hash_oracle_sample(wl, s, ell, rows=1_000_000):
    """The oracle's hash sketch (as it stands, one thread) on the first `rows` rows."""
    import fdgen
    import oracle
    cfgname = WORKLOADS[wl][0]
    w = fdgen.config(cfgname)
    nr = min(rows, w.n)
    A = fdgen.host_rows(w, 0, nr)
    t0 = time.perf_counter()
    oracle.hash_sketch(A, ell, s=s, seed=0)
    dt = time.perf_counter() - t0
    return {"value": nr / dt, "unit": "rows/s", "cores": 1, "kind": "oracle",
            "sample": f"first {nr} rows of {wl}, fp64 oracle hash sketch, one thread, {dt:.1f} s"}


def run_hash(args):
    import torch
    import torch.distributed as dist

    import fdgen
    import paper_1501_06561_b200 as fd
    from paper_1501_06561_b200.dist import local_range, reduce_hash

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    cfgname, ell, _, _ = WORKLOADS[wl]
    s = HASH_S[args.variant]
    w = fdgen.config(cfgname)
    r0, r1 = local_range(w.n, rank, world)
    nloc = r1 - r0
    gen = fdgen.DeviceGenerator(w, device=dev)
    A = torch.empty((nloc, w.d), dtype=torch.float32, device=dev)
    gen.fill(A, r0)
    B = torch.zeros((ell, w.d), dtype=torch.float64, device=dev)
    nws = fd.lib().fd_hash_workspace_bytes(w.d, ell)
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        B.zero_()
        fd.check(fd.lib().fd_hash_sketch(A.data_ptr(), nloc, A.stride(0), w.d, ell, s, 0, r0, B.data_ptr(),
                                         ws.data_ptr(), nws, stream.cuda_stream))
        reduce_hash(B)                # the sketch is linear: the merge is a sum
        return B

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    kern_ms = 0.0
    for _ in range(args.steps):
        B.zero_()
        k0.record(stream)
        fd.check(fd.lib().fd_hash_sketch(A.data_ptr(), nloc, A.stride(0), w.d, ell, s, 0, r0, B.data_ptr(),
                                         ws.data_ptr(), nws, stream.cuda_stream))
        k1.record(stream)
        reduce_hash(B)
        k1.synchronize()
        kern_ms += k0.elapsed_time(k1)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = w.n / (ms_step / 1e3)
    pk = peaks()
    kms = kern_ms / args.steps
    bytes_launch = nloc * w.d * 4.0 + 2.0 * fd.lib().fd_hash_workspace_bytes(w.d, ell) + 2.0 * ell * w.d * 8
    roof = {"bound": "hbm", "achieved": bytes_launch / (kms / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "kernel": "hash_kernel+hash_reduce_kernel",
            "algorithmic_bytes": "n d 4 (read A) + 2 x partials (write + read, fp64) + B read/write",
            "traffic": None, "peak_source": f"hbm_gbs {pk['source']}", "ms_per_launch": kms}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # measured DRAM traffic of one launch (ncu --set full capture, c4 only, one GPU)
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if wl == "c4" and world == 1 and os.path.exists(traffic_file):
        with open(traffic_file) as f:
            tr = json.load(f).get(f"hash_kernel_s{s}")
        if tr:
            roof["traffic"] = tr["bytes_per_launch_captured"]
            roof["traffic_source"] = tr["source"]
    # error of the hash sketch (GPU evaluator, outside the timed region)
    from paper_1501_06561_b200.dist import dist_cov_err
    Bf = B.to(torch.float32)
    ce = dist_cov_err(A, Bf, proj_k=10)
    e2e = None
    if not args.no_e2e:
        chunk = 1 << 18
        Ah = torch.empty((nloc, w.d), dtype=torch.float32, pin_memory=True)
        Ah.copy_(A)
        del A
        torch.cuda.empty_cache()
        bufs = [torch.empty((chunk, w.d), dtype=torch.float32, device=dev) for _ in range(2)]
        copy_s = torch.cuda.Stream(dev)
        done = [torch.cuda.Event() for _ in range(2)]
        copied = [torch.cuda.Event() for _ in range(2)]

        def e2e_step():
            # chunk k+1 is copied (copy stream) while chunk k is hashed (compute stream)
            B.zero_()
            for ci, a in enumerate(range(0, nloc, chunk)):
                b = min(nloc, a + chunk)
                k = ci & 1
                with torch.cuda.stream(copy_s):
                    if ci >= 2:
                        copy_s.wait_event(done[k])
                    bufs[k][: b - a].copy_(Ah[a:b], non_blocking=True)
                    copied[k].record(copy_s)
                stream.wait_event(copied[k])
                fd.check(fd.lib().fd_hash_sketch(bufs[k].data_ptr(), b - a, w.d, w.d, ell, s, 0, r0 + a,
                                                 B.data_ptr(), ws.data_ptr(), nws, stream.cuda_stream))
                done[k].record(stream)
            reduce_hash(B)
            return B.cpu()

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ks = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(ks):
            e2e_step()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        sec = float(el.item()) / ks
        e2e = {"value": w.n / sec, "unit": "rows/s", "h2d_bytes_per_step": int(w.n * w.d * 4),
               "d2h_bytes_per_step": int(ell * w.d * 8 * world), "steps": ks,
               "note": "wall clock: pinned host rows -> H2D chunks (2 streams) -> fd_hash_sketch -> D2H of B"}
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 accumulation of f32 rows", "data": "synthetic (seeded fdgen, generated on device)",
        "config": {"workload": f"{wl}: n={w.n} d={w.d} ell={ell}, {args.variant} (s={s}), seed 0",
                   "n": w.n, "d": w.d, "ell": ell, "variant": args.variant, "s": s,
                   "parallelism": f"rows dp{world} + all_reduce(B)",
                   "l2": "inputs larger than L2 (A is streamed from HBM every step)"},
        "roofline": roof, "gpu_launches": 2 * args.steps,
        "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"]},
        "cov_err": ce["err"], "cov_err_lmin": ce["lmin"], "proj_err_k10": ce.get("proj_err"), "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = hash_oracle_sample(wl, s, ell)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default=None)
    ap.add_argument("--alpha", type=float, default=0.2, help="alpha of the alpha-FD variants")
    ap.add_argument("--shards", type=int, default=None, help="P_total shard streams (default: the workload's)")
    ap.add_argument("--ell", type=int, default=None, help="sketch size (default: the workload's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 is below the timing rules", file=sys.stderr)
    if args.variant in HASH_S:
        if args.impl == "reference":
            rank, _, _ = dist_env()
            if rank == 0:
                res = hash_oracle_sample(args.workload, HASH_S[args.variant], WORKLOADS[args.workload][1])
                print(json.dumps({"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "rows/s",
                                  "n_gpus": args.gpus, "steps": 1, "warmup": 0, "higher_is_better": True,
                                  "dtype": "f64", "data": "synthetic", "cpu_baseline": res,
                                  "e2e": {"value": res["value"], "unit": "rows/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            return 0
        return run_hash(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
