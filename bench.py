"""Benchmark: one step = one full thin SVD (Gram + Jacobi + U) of one
synthetic matrix of a BASELINE.json configuration, device-resident.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

The default workload is c4 (m=2^26, n=128, fp32 working, Gram in fp64,
Gaussian A): the largest single-GPU configuration of BASELINE.json's
binary32 path, the one its north_star quotes the >= 60 % roofline and the
>= 6x 8-GPU scaling targets on. For N>1 the driver launches one process per
GPU (torchrun); the 2^26 rows are block-sharded (strong scaling), each rank
forms its partial Gram, the partials meet in ONE NCCL all-gather followed by
the reference's fixed tree over ranks inside the library, the Jacobi is
replicated and U stays rank-local. (c2 runs weak scaling: 2^20 rows per
rank.) Rank 0 prints ONE JSON line.

`--impl reference` times the reference's own CPU implementation (the
unmodified reference compiled in place, oracle/_ref; the C restatement
oracle/_port when the reference has no path, i.e. the double-double
configs) on the host cores, on a row sample sized so the whole run stays
within a few minutes. That arm imports only oracle/ and workloads.py, never
the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "thin-SVD time & effective TFLOP/s (Gram+AV) at 1/2/4/8 B200; % of roofline"
UNIT = "TFLOP/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def flops(m: int, n: int):
    """Algorithmic work per SVD: upper-triangle SYRK and AV."""
    return float(m) * n * (n + 1), 2.0 * m * n * n


# fp64 FMA-pipe rate (DFMA, profiles/r01_microbench.txt): the double-double
# kernels are bound by fp64 instruction issue, one operation per lane-cycle
DFMA_TFLOPS = 34.2


EIG = {"twosided": 0, "gramchol": 1, "onesided": 2}
EIG_NAME = {0: "TwoSidedJacobi", 1: "GramCholSvd", 2: "OneSidedJacobiOnGram"}


def config_dict(cfg, world: int, eig: int = 0):
    """The workload both arms report (the reference arm times a row sample of
    it, named in its cpu_baseline.sample)."""
    m_global = cfg.m * world if cfg.name == "c2" else cfg.m
    m_local = cfg.m if cfg.name == "c2" else -(-cfg.m // world)
    esz = 4 if cfg.working == "f32" else 8
    return {"workload": cfg.name, "m": m_global, "n": cfg.n, "working": cfg.working,
            "gram": "fp64" if cfg.working == "f32" else "double-double",
            "l2": f"inputs larger than L2 (A = {m_local * cfg.n * esz / 2**20:.0f} MiB per GPU > 126 MB)",
            "parallelism": f"rows{world}", "eigensolver": EIG_NAME[eig]}


OZ_PRODUCTS = 66                               # digit products p + q <= 12 of 11 digits (gram_ozaki.cu)
I8_TOPS = 2 * 128 * 256 * 32 / 128 * 148 * 1.965e9 / 1e12  # 4.77 POPS (umma_i8 probe)


K1Z_MMAS_PER_CHUNK = 12                        # 2 CTAs x 6 M128 N128 K32 int8 digit products per 32-row chunk (gram_ozaki32.cu; issued as 5 + 4 MMAs)
NCU_NAME = {("gram", 0): "gram_f32_diag", ("gram", 1): "gram_f32_ozaki", ("gram", 2): "gram_f64_dd",
            ("gram", 3): "gram_dd_ozaki", ("compute_u", 0): "av_kernel", ("compute_u", 1): "av_tc_tmem_f32",
            ("compute_u", 2): "av_dmma_f64"}
GRAM_KERNELS = {0: "K1 gram_f32_diag/offdiag (DMMA)", 1: "K1z gram_f32_ozaki (tcgen05 kind::i8, TMA)",
                2: "K2 gram_f64_dd (Dot2, fp64 pipe)", 3: "K2z gram_dd_ozaki (tcgen05 kind::i8) + ozaki_slice/colexp"}
AV_KERNELS = {0: "av_kernel (fp32 SIMT)", 1: "av_tc_tmem_f32 (tcgen05, fp16 pieces: A x2, W x3)", 2: "av_dmma_f64 (DMMA)"}


def phase_rooflines(cfg, m_local, n, med, fp64_peak, hbm, info):
    """Roofline of every pipeline phase of one SVD on one GPU, each against
    the bound of the kernel the plan actually ran (info.gram_kernel /
    info.av_kernel, reported by the library):

    gram K1 : m n (n+1) flops on the DMMA pipe
    gram K1z: 12 int8 digit products (M = N = 128, K = 32; issued as 9 MMAs,
              three of them N = 256) per 32-row chunk = 12 x 2 x 128 x 128
              ops per row, against the int8 tensor peak; also
              m n 4 bytes of A against HBM (hbm_frac)
    gram K2 : m n (n+1)/2 multiply-adds x 10 fp64 operations (c_dd = 10,
              SURVEY.md §8(d)) against the DFMA issue rate
    gram K2z: 66 int8 digit products per multiply-add on the int8 tensor cores
    eigen   : two-sided Jacobi, latency bound (see `jacobi`); 18 n flops per
              rotation against fp64 peak for reference only
    U  f32  : read A + write U (2 m n 4 bytes) against HBM (K7 on the tensor
              cores, far from their bf16 bound)
    U  f64  : 2 m n^2 flops on the DMMA pipe (av_dmma_f64)
    """
    out = {}
    gk = int(getattr(info, "gram_kernel", -1))
    ak = int(getattr(info, "av_kernel", -1))
    t_g = med["gram"] * 1e-3
    if gk == 1:
        ops = float(m_local) * K1Z_MMAS_PER_CHUNK * 2 * 128 * 128
        a = ops / t_g / 1e12
        bw = m_local * n * 4 / t_g / 1e9
        out["gram"] = {"kernel": GRAM_KERNELS[1], "bound": "tensor", "achieved": a, "peak": I8_TOPS,
                       "unit": "TOPS", "frac": a / I8_TOPS,
                       "peak_source": "tcgen05 kind::i8 probe: one M128 N256 K32 MMA per 128 cycles per SM "
                                      "(tools/microbench/umma_i8.cu, profiles/r01_umma_i8.txt) x 148 SMs x 1965 MHz",
                       "algorithmic": "12 x 2 x 128 x 128 int8 ops per row of A (2 CTA groups x 6 digit products "
                                      "per 32-row chunk, issued as 5 + 4 MMAs)",
                       "hbm_achieved_gbs": bw, "hbm_frac": bw / hbm,
                       "fp64_equivalent_tflops": m_local * n * (n + 1) / t_g / 1e12}
    elif gk == 0:
        a = m_local * n * (n + 1) / t_g / 1e12
        out["gram"] = {"kernel": GRAM_KERNELS[0], "bound": "tensor", "achieved": a,
                       "peak": fp64_peak, "unit": "TFLOP/s", "frac": a / fp64_peak,
                       "peak_source": "live DMMA m8n8k4 probe (MEASURED_PEAKS.json has no fp64 figure)",
                       "algorithmic": "m*n*(n+1) flops per SVD"}
    elif gk == 3:
        ops = 2.0 * OZ_PRODUCTS * m_local * n * (n + 1) / 2
        a = ops / t_g / 1e12
        out["gram"] = {"kernel": GRAM_KERNELS[3], "bound": "tensor",
                       "achieved": a, "peak": I8_TOPS, "unit": "TOPS", "frac": a / I8_TOPS,
                       "peak_source": "tcgen05 kind::i8 probe: one M128 N256 K32 MMA per 128 cycles per SM "
                                      "(tools/microbench/umma_i8.cu, profiles/r01_umma_i8.txt) x 148 SMs x 1965 MHz",
                       "algorithmic": "2 x 66 int8 digit products x m x n(n+1)/2 (upper triangle) per SVD",
                       "dd_equivalent_tops": m_local * n * (n + 1) / 2 * 10 / t_g / 1e12}
    else:
        ops = m_local * n * (n + 1) / 2 * 10
        peak = DFMA_TFLOPS / 2
        a = ops / t_g / 1e12
        out["gram"] = {"kernel": GRAM_KERNELS.get(gk, "K2 gram_f64_dd"), "bound": "fp64", "achieved": a,
                       "peak": peak, "unit": "Tops/s", "frac": a / peak,
                       "peak_source": "DFMA issue rate (profiles/r01_microbench.txt 34.2 TFLOP/s / 2)",
                       "algorithmic": "c_dd = 10 fp64 ops per multiply-add, m*n*(n+1)/2 multiply-adds"}
    t_u = med["compute_u"] * 1e-3
    if cfg.working == "f32":
        b = 2.0 * m_local * n * 4 / t_u / 1e9
        out["compute_u"] = {"kernel": AV_KERNELS.get(ak, "av"), "bound": "hbm", "achieved": b, "peak": hbm,
                            "unit": "GB/s", "frac": b / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                            "algorithmic": "2*m*n*4 bytes (read A, write U) per SVD"}
    else:
        f = 2.0 * m_local * n * n / t_u / 1e12
        out["compute_u"] = {"kernel": AV_KERNELS.get(ak, "av_dmma_f64 (DMMA)"), "bound": "tensor", "achieved": f,
                            "peak": fp64_peak, "unit": "TFLOP/s", "frac": f / fp64_peak,
                            "peak_source": "live DMMA m8n8k4 probe",
                            "algorithmic": "2*m*n^2 flops per SVD"}
    out["gram"]["ncu_kernel"] = NCU_NAME.get(("gram", gk))
    out["compute_u"]["ncu_kernel"] = NCU_NAME.get(("compute_u", ak))
    jf = 18.0 * n * info.rotations / (med["eigen"] * 1e-3) / 1e12
    out["eigen"] = {"kernel": "jacobi_smem / jacobi_kernel", "bound": "latency", "achieved": jf,
                    "peak": DFMA_TFLOPS, "unit": "TFLOP/s", "frac": jf / DFMA_TFLOPS,
                    "algorithmic": "18*n flops per rotation; one CTA, ~n/2 rotations per barrier round"}
    return out


def latency_probe():
    """Measured latency floors (tools/microbench/rot_latency.cu on the B200,
    committed as profiles/r02_latency_probe.json): cycles of one dependent
    fp64 rotation (stop test + rotation), one 512-thread __syncthreads
    hand-off, one 148-CTA grid barrier (the solver's arrival counter)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_latency_probe.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def jacobi_latency(n: int, info, eigen_ms: float, dd: bool, clock_mhz: float = 1965.0):
    """The two-sided Jacobi against its latency floor: every parallel round is
    one dependent rotation evaluation followed by one hand-off (a CTA barrier
    for the single-CTA solver, n <= 128 fp64 / <= 100 dd; a grid barrier for
    the cooperative solver), so T_floor = rounds x (rotation chain +
    barrier). The eigen phase also holds the V replay / finish kernels."""
    rounds = int(getattr(info, "rounds", 0) or 0)
    out = {"kernel": "jacobi_smem" if n <= (100 if dd else 128) else "jacobi_kernel (cooperative grid)",
           "bound": "latency", "sweeps": int(info.sweeps), "rounds": rounds, "eigen_ms": eigen_ms}
    if rounds <= 0:
        return out
    cyc = eigen_ms * 1e-3 * clock_mhz * 1e6 / rounds
    out["cycles_per_round"] = cyc
    pr = latency_probe()
    chain = pr.get("rotation_chain_cycles")
    bar = pr.get("grid_sync_cycles") if out["kernel"].startswith("jacobi_kernel") else pr.get("syncthreads_cycles")
    if chain and bar:
        floor = chain + bar
        out["floor_cycles_per_round"] = floor
        out["floor_ms"] = rounds * floor / (clock_mhz * 1e3)
        out["frac"] = floor / cyc
        out["floor_definition"] = ("rounds x (one dependent fp64 rotation chain + one barrier hand-off), "
                                   "profiles/r02_latency_probe.json" + (" (fp64 chain: a lower bound for the dd solver)"
                                                                        if dd else ""))
    return out


def traffic_for(kernel: str, config: str):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    `kernel` (its ncu function name) from a committed ncu --set full capture
    (profiles/r02_traffic.json, else r01), or None."""
    for f in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", f)) as fh:
                t = json.load(fh)
        except (OSError, ValueError):
            continue
        v = t.get(config, {}).get(kernel)
        if v is not None:
            return v
    return None


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def _sample_rows(cfg, fn_for, budget_s: float, runs: int):
    """Largest power-of-two row count (<= cfg.m, >= 2^12) whose run fits
    budget_s / runs seconds, from one timed calibration run on 2^14 rows
    (the CPU path is linear in m at fixed n)."""
    m0 = min(cfg.m, 1 << 14)
    fn = fn_for(m0)
    fn()  # page-in / thread-pool start-up
    t0 = time.perf_counter()
    fn()
    t = max(time.perf_counter() - t0, 1e-4)
    per_run = budget_s / max(runs, 1)
    m_s = m0
    while m_s * 2 <= cfg.m and (m_s * 2) / m0 * t <= per_run:
        m_s *= 2
    return m_s


def run_reference(args, cfg, budget_s: float = 150.0):
    """CPU reference arm: rank 0 only, all host threads, a row sample of the
    workload sized so warm-up + timed runs take about budget_s seconds."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    import workloads as inputs

    cores = os.cpu_count() or 1
    n = cfg.n
    eig = EIG[args.eig]
    runs = args.steps + args.warmup
    what = f"mp_thin_svd {EIG_NAME[eig]}"
    if cfg.working == "f32":
        lib = pyoracle.Ref() if pyoracle.ref_available() else pyoracle.Port()
        kind = "reference" if pyoracle.ref_available() else "port"

        def fn_for(m_s):
            a = inputs.make(cfg, seed=1, m=m_s)
            return lambda: lib.thin_svd(a, threads=cores, choice=eig)
        flops_fn = flops
    elif cfg.n <= 256:
        # no reference path for binary64 input (thinsvd.cpp:52-53): the
        # restated double-double oracle, whole pipeline (dd Gram + dd Jacobi + U)
        lib, kind = pyoracle.Port(), "port"
        what = "restated double-double thin SVD (dd Gram + dd two-sided Jacobi + U), not reference code"

        def fn_for(m_s):
            a = inputs.make(cfg, seed=1, m=m_s)
            return lambda: lib.thin_svd_f64dd(a, threads=cores)
        flops_fn = flops
    else:
        # c5 (n = 1024): the restated dd Jacobi alone is hours of CPU time
        # (O(n^3) double-double work per sweep, ~45 sweeps), so the sample
        # times the Gram-phase oracle only - the dd Gram of the reference's
        # test support (dd.cpp:75-88), restated - and prices it with the
        # Gram flops alone (the metric's F_gram part)
        lib, kind = pyoracle.Port(), "port"
        what = "restated double-double Gram only (dd_gram, dd.cpp:75-88), not reference code; Jacobi and U not run"

        def fn_for(m_s):
            a = inputs.make(cfg, seed=1, m=m_s)
            return lambda: lib.dd_gram(a, threads=cores)
        flops_fn = lambda m, nn: (float(m) * nn * (nn + 1), 0.0)  # noqa: E731
    m_s = _sample_rows(cfg, fn_for, budget_s, runs)
    fn = fn_for(m_s)
    for _ in range(args.warmup):
        fn()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    fg, fa = flops_fn(m_s, n)
    value = (fg + fa) / t / 1e12
    sample = (f"{cfg.name} distribution with m={m_s} rows (of {cfg.m}; the largest power of two fitting "
              f"~{budget_s:.0f} s of CPU for the whole run), n={n}; median of {args.steps} after {args.warmup} "
              f"warm-up; {what}; {cores} threads")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if cfg.name == "c2" else "strong", "vs_baseline": None,
        "dtype": "f64" if cfg.working == "f32" else "f64x2",
        "data": "synthetic (seeded, BASELINE.json distribution)",
        "config": dict(config_dict(cfg, args.gpus, eig), sample_rows=m_s),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def cpu_baseline(cfg, eig="twosided"):
    """Reported baseline (not the target): the reference arm's measurement
    on a smaller sample (~25 s of CPU work) so the default run stays short."""
    ns = argparse.Namespace(steps=3, warmup=1, gpus=1, eig=eig)
    line = run_reference(ns, cfg, budget_s=25.0)
    return line["cpu_baseline"] if line else None


# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2603_11953_b200 as M
    import workloads as inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    n = cfg.n
    if cfg.name == "c2" or world == 1:
        m_local = cfg.m  # weak scaling for c2; the full config at N=1
    else:
        base, extra = divmod(cfg.m, world)
        m_local = base + (1 if rank < extra else 0)
    m_global = m_local * world if (cfg.name == "c2" or world == 1) else cfg.m
    working = M.Precision.WORKING if cfg.working == "f32" else M.Precision.HIGHER
    esz = 4 if cfg.working == "f32" else 8

    comm = None
    if world > 1:
        uid = [M.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = M.Comm(uid[0], world, rank)

    def allreduce_cpu(t):
        c = t.cpu()
        dist.all_reduce(c)
        return c.to(t.device)

    a_t = inputs.device_make(cfg, seed=1, m=m_local, device=dev, rank=rank,
                             allreduce=allreduce_cpu if world > 1 else None)  # (n, m) = column-major m x n
    u_t = torch.empty_like(a_t)
    sig_t = torch.empty(n, dtype=torch.float64, device=dev)
    v_t = torch.empty((n, n), dtype=a_t.dtype, device=dev)
    plan = M.Plan(m_local, n, working, comm)
    eig = EIG[args.eig]
    if eig:
        if cfg.working != "f32":
            raise SystemExit("--eig gramchol/onesided: binary32 configs only (the reference has no fp64 path)")
        plan.set_eigensolver(eig)
    # a dedicated (non-legacy) stream: the plan enqueues every kernel on it and
    # the CUDA events below are recorded on the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0
    torch.cuda.synchronize()

    def step():
        plan.execute(a_t.data_ptr(), m_local, u_t.data_ptr(), m_local, sig_t.data_ptr(), v_t.data_ptr(), sptr)

    for _ in range(args.warmup):
        step()
    info = plan.wait()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # timed region: barrier + synchronize on both sides, device events on the
    # plan's stream, max over ranks below
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    phase = {"gram": [], "eigen": [], "compute_u": []}
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = e0.elapsed_time(e1)
    # per-phase device times (CUDA events inside the library, same stream),
    # from separately synchronised steps so each phase is isolated
    for _ in range(min(args.steps, 5)):
        step()
        inf = plan.wait()
        phase["gram"].append(inf.ms_gram)
        phase["eigen"].append(inf.ms_eigen)
        phase["compute_u"].append(inf.ms_compute_u)
    clk = clocks.stop()
    info = plan.wait()
    if info.status != 0:
        raise RuntimeError(f"device pipeline status {info.status}")
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # full-size validation of the factorisation just timed, on the device
    # (SURVEY.md §8(f)-2): max row-wise backward error (max over ranks), the
    # north_star orthogonality gates ||U^T U - I||_F (U^T U by the plan's own
    # Gram stage, exchange included, so it is global over ranks) and
    # ||V^T V - I||_F, and for c5 sigma against the prescribed values
    bw = M.backward_error_device(a_t.T, u_t.T, sig_t, v_t.T, stream)
    u_w = 2.0 ** -24 if cfg.working == "f32" else 2.0 ** -53
    orth_u = plan.orth_error(u_t.data_ptr(), m_local, sptr)
    v64 = v_t.double().cpu().numpy().T  # (n, n) column-major V
    orth_v = float(np.linalg.norm(v64.T @ v64 - np.eye(n)))
    validation = {"rowwise_backward_error": bw.max_rel, "skipped_rows": bw.skipped_rows,
                  "unit_roundoff": u_w,
                  "definition": "max_i ||(U diag(s) V^T - A)(i,:)|| / ||A(i,:)||, binary64 (metrics.cpp:40-70)",
                  "orth_u": orth_u, "orth_v": orth_v, "orth_gate": 10.0 * n * u_w,
                  "orth_definition": "||Q^T Q - I||_F in binary64 (dense.cpp:250-272); gate 10*n*u (north_star)"}
    if cfg.kind == "prescribed":
        want = 10.0 ** (-cfg.decades * np.arange(n) / max(n - 1, 1))
        got = sig_t.cpu().numpy()
        validation["sigma_vs_prescribed_max_rel"] = float(np.max(np.abs(got - want) / want))
        validation["sigma_note"] = ("A = U0 diag(sigma) V0^T is formed in binary64, which perturbs sigma_i by "
                                    "about u*sigma_1/sigma_i (up to ~1e-6 relative at sigma_n = 1e-10)")
    if world > 1:
        t = torch.tensor([bw.max_rel, float(bw.skipped_rows)], dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        validation["rowwise_backward_error"], validation["skipped_rows"] = float(t[0]), int(t[1])

    fg, fa = flops(m_global, n)
    value = (fg + fa) / (ms * 1e-3) / 1e12
    med = {k: statistics.median(v) for k, v in phase.items()}

    # --- e2e through the reference-facing C ABI with host buffers -----------
    e2e = None
    if world == 1:
        # the public host-buffer API on this GPU only (MPSVD_DEVICES: it would
        # otherwise shard over every visible GPU of the node)
        os.environ["MPSVD_DEVICES"] = str(local)
        host = M.Matrix(m_local, n, working)
        # A straight into the page-locked host matrix: its (n, m) transpose
        # view is the same column-major memory as a_t
        torch.from_numpy(host.numpy().T).copy_(a_t)
        # free the device-resident arm before the API allocates its own buffers
        del plan, a_t, u_t, v_t, sig_t
        torch.cuda.empty_cache()
        call = (lambda h: M.mp_thin_svd(h, choice=eig)) if cfg.working == "f32" else M.mp_thin_svd_f64
        r = call(host)  # warm: plan, device buffers, pinned result buffers
        del r
        reps = 5
        t_e2e = 0.0
        for _ in range(reps):
            t0 = time.perf_counter()
            r = call(host)
            t_e2e += time.perf_counter() - t0
            times = r.times
            del r  # result buffers go back to the pinned pool
        t_e2e /= reps
        e2e = {"value": (fg + fa) / t_e2e / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": m_local * n * esz,
               "d2h_bytes_per_step": m_local * n * esz + n * n * esz + n * 8,
               "ms_per_step": t_e2e * 1e3,
               "phase_s": {"gram": times.gram, "eigen": times.eigen, "compute_u": times.compute_u,
                           "overlap": times.overlap, "total": times.total}}
    else:
        # N > 1: the multi-GPU public API (Plan + Comm, C ABI mpsvd_plan_*)
        # with page-locked host buffers per rank: H2D of the rank's rows of A,
        # the pipeline (one NCCL exchange inside), D2H of U, sigma and V;
        # wall time per step, max over ranks
        h_a = torch.empty(a_t.shape, dtype=a_t.dtype, pin_memory=True)
        h_a.copy_(a_t)
        h_u = torch.empty(a_t.shape, dtype=a_t.dtype, pin_memory=True)
        h_s = torch.empty(n, dtype=torch.float64, pin_memory=True)
        h_v = torch.empty((n, n), dtype=a_t.dtype, pin_memory=True)
        reps = 5
        t_e2e = 0.0
        for i in range(reps + 1):
            dist.barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                a_t.copy_(h_a, non_blocking=True)
                step()
                h_u.copy_(u_t, non_blocking=True)
                h_s.copy_(sig_t, non_blocking=True)
                h_v.copy_(v_t, non_blocking=True)
            stream.synchronize()
            if i > 0:  # first repetition is a warm-up
                t_e2e += time.perf_counter() - t0
        t_e2e /= reps
        tt = torch.tensor([t_e2e], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
        e2e = {"value": (fg + fa) / t_e2e / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": m_local * n * esz,
               "d2h_bytes_per_step": m_local * n * esz + n * n * esz + n * 8,
               "ms_per_step": t_e2e * 1e3, "path": "mpsvd_plan_* with an NCCL communicator, per-rank bytes"}

    if rank != 0:
        return None

    pk = peaks()
    fp64_peak = M.fp64_peak_tflops(local)
    hbm = pk.get("hbm_gbs", 6650.0)
    # per-phase rooflines: algorithmic work per launch over
    # the phase's CUDA-event time on the plan's stream. The headline
    # `roofline` is the dominant throughput kernel of the Gram+AV pair (the
    # north_star's roofline scope), each against its own bound: K1 on the
    # DMMA pipe, K2z on the int8 tensor cores, K7 f32 on HBM, K7 f64 on
    # DMMA. The Jacobi is latency-bound and reported beside it (`jacobi`).
    phases = phase_rooflines(cfg, m_local, n, med, fp64_peak, hbm, info)
    dom = max(("gram", "compute_u"), key=lambda k: med[k])
    roof = dict(phases[dom])
    roof["phase"] = dom
    roof["traffic"] = traffic_for(roof.get("ncu_kernel") or "", cfg.name)
    if roof.get("ncu_kernel") == "gram_f32_ozaki" and roof["traffic"]:
        # the ncu capture is one of the Gram's 16 range launches (one per logical block)
        roof["traffic_note"] = ("DRAM bytes of ONE K1z range launch of c4 at N = 1 (2^22 rows, algorithmic 2^22 x 128 x 4 B = "
                                "2.147e9); a Gram is 16 such launches")
    jac = jacobi_latency(n, info, med["eigen"], cfg.working != "f32")
    # north_star roofline for the whole Gram+AV pair
    t_hbm = 2.0 * m_global / world * n * esz / (hbm * 1e9)
    t_cmp = (fg + fa) / world / (fp64_peak * 1e12) if cfg.working == "f32" else (fg * 5 + fa) / world / (fp64_peak * 1e12)
    t_roof = max(t_hbm, t_cmp)
    gram_av_ms = med["gram"] + med["compute_u"]
    floor_ms = {}
    for ph in ("gram", "compute_u"):
        r = phases[ph]
        t_ach = med[ph]
        t_unit = t_ach * r["achieved"] / r["peak"]           # the kernel's work at its unit's peak
        t_bytes = (m_local * n * esz * (1 if ph == "gram" else 2)) / (hbm * 1e9) * 1e3
        floor_ms[ph] = max(t_unit, t_bytes)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if cfg.name == "c2" else "strong", "vs_baseline": None,
        "dtype": "f64" if cfg.working == "f32" else "f64x2",
        "data": "synthetic (seeded torch generator, BASELINE.json distribution)",
        "config": config_dict(cfg, world, eig),
        "phase_ms": med,
        "roofline": roof,
        "roofline_phases": phases,
        "jacobi": jac,
        "svd_roofline": {"definition": "max(2*m*n*s/HBM, F_gram/P_gram + F_AV/P_fp64) (north_star)",
                         "t_roof_ms": t_roof * 1e3, "gram_plus_av_ms": gram_av_ms,
                         "frac": (t_roof * 1e3) / gram_av_ms if gram_av_ms > 0 else None,
                         "p_fp64_tflops": fp64_peak,
                         "per_kernel_floor_ms": floor_ms,
                         "per_kernel_frac": sum(floor_ms.values()) / gram_av_ms if gram_av_ms > 0 else None,
                         "per_kernel_definition": "each of the Gram and U kernels at the floor of the resource it "
                                                  "runs on (the slower of its algorithmic work at that unit's "
                                                  "peak and its HBM bytes at measured HBM), summed"},
        "gpu_launches": info.kernel_launches * args.steps,
        "clocks": clk,
        "e2e": e2e,
        "sweeps": info.sweeps,
        "validation": validation,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.eig)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eig", default="twosided", choices=list(EIG),
                    help="mp_thin_svd spectral branch (GramCholSvd / OneSidedJacobiOnGram: binary32 configs)")
    args = ap.parse_args()
    from workloads import CONFIGS

    cfg = CONFIGS[args.config]
    line = run_reference(args, cfg) if args.impl == "reference" else run_ours(args, cfg)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
