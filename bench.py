"""Benchmark of the B200 Kronecker space-time heat solve (BASELINE.json metric).

Workload: config 3 -- 2D heat, Q1 on a 1023 x 1023 interior grid, n_t = 1024 (1.07e9 FP64
unknowns), full-rank F ~ U[-1,1] from the seeded counter generator.  One step = one full
solve F -> U (solve_projected_heat_with in tensor form: DMMA transforms + modal scan).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* value      : unknowns/s with F and U resident in HBM (CUDA events on the plan stream,
               barrier + synchronize on both sides, max over ranks).
* e2e        : unknowns/s through the public host-buffer API (stkg_heat_solve_host) with
               the H2D of F and the D2H of U (pinned host memory) inside the timed region.
* roofline   : dominant kernel = the axis-transform kernel of the headline backend:
               --transform dst (default): FP64 Stockham-FFT sine transforms, HBM-bound,
               achieved = 16 B/unknown per axis pass / mean launch time vs measured HBM BW;
               --transform dense: DMMA GEMMs, achieved = 2n flop/unknown per pass / mean
               launch time vs the measured DMMA FP64 peak.  Launch times come from CUDA
               events around every launch on the plan stream.  The other backend is timed
               too and reported under "alt_path".
* cpu_baseline / --impl reference : the oracle port of solve_projected_heat_with
               (oracle/oracle.py::heat_decoupled, numpy + multithreaded BLAS) on a bounded
               causal prefix of the same workload, on this host's cores.
N > 1 runs independent replicas (in-scope multi-GPU is replicas only).
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "space-time unknowns solved/sec (FP64) and % of HBM/FP64 roofline vs CPU ref"
UNIT = "unknowns/s"
# Measured on this pool's B200 (profiles/r01_fp64_peak.txt): DMMA m16n8k16 sustained.
FP64_PEAK_TFLOPS = 37.11
FP64_PEAK_SOURCE = "measured DMMA (mma.sync f64) sustained, profiles/r01_fp64_peak.txt"


def _hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth on this pool's B200s)."""
    try:
        v = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6553.9, "fallback: MEASURED_PEAKS.json hbm_gbs of round 1 (file unreadable)"


HBM_GBS, HBM_SOURCE = _hbm_peak()
CPU_SAMPLE_STEPS = 320  # causal prefix of cfg3 time slices for the CPU leg (~10 s)
REF_MAX_CHUNK = 64  # time slices per oracle call in the streamed reference arm
# precond = 4 GEMMs of 2 n_h n_h n_t' flop (TwoTermPrecond::solve) + WaveOperator ~84 flop/unknown
WAVE_FLOP_PER_PCG_ITER = lambda nh, ntb: 4 * 2.0 * nh * nh * ntb + 84.0 * nh * ntb  # noqa: E731


def loaded_native_libs():
    """Shared objects of this repository (and any torch extension) mapped into this process:
    the evidence that the reference arm runs without the product library."""
    libs = set()
    try:
        for ln in Path("/proc/self/maps").read_text().splitlines():
            parts = ln.split()
            if parts and parts[-1].endswith(".so") or ".so." in (parts[-1] if parts else ""):
                path = parts[-1]
                if path.startswith(str(ROOT)) or "torch_extensions" in path:
                    libs.add(os.path.relpath(path, ROOT) if path.startswith(str(ROOT)) else path)
    except Exception:
        pass
    return sorted(libs)


def fft_flop_per_unknown(n: int, half: bool) -> float:
    """Executed flops of one DST-I axis pass per unknown (complex FFT of length L per vector
    pair, 5 L log2 L / 2 per vector, spread over n entries)."""
    L = (n + 1) if half else 2 * (n + 1)
    return 5.0 * L * np.log2(L) / 2.0 / n


def half_kernels(cfg) -> bool:
    """Whether the plan runs the half-length DST kernels (heat.cu::dst_pass: 2D/3D plans
    with N = n + 1 a power of two in [16, 1024])."""
    N = cfg.n + 1
    return (cfg.ndim >= 2 and 16 <= N <= 1024 and N & (N - 1) == 0
            and os.environ.get("STKG_DST_HALF", "1") != "0")


def workload_config(cfg):
    """The `config` object both arms print for a heat workload (identical keys and values)."""
    return {"workload": cfg.name, "unknowns_per_solve": cfg.unknowns, "ndim": cfg.ndim,
            "n": cfg.n, "nt": cfg.nt, "load_rank": cfg.rank or "full", "seed": 0,
            "l2_flush": "inputs larger than L2 (F, U 8.6 GB each)" if cfg.unknowns * 8 > 2**30
            else "none"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def max_over_ranks(x: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device times are combined by the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(unknowns_per_step: int, steps: int, world: int, ms_max: float) -> float:
    """Whole-job throughput: every replica solved `steps` systems in at most ms_max."""
    return world * unknowns_per_step * steps / (ms_max / 1e3)


def e2e_slices(cfg, world: int) -> int:
    """Time slices of the end-to-end leg: all of n_t unless the ranks on this node would
    not fit their pinned F and U copies (2 x 8 B per unknown each) in ~60% of the available
    host memory, in which case a causal prefix is solved (e2e throughput is linear in n_t;
    the JSON records the slice count)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        return cfg.nt
    local = int(os.environ.get("LOCAL_WORLD_SIZE", world) or 1)
    budget = 0.6 * avail / max(local, 1)
    per_slice = 2 * cfg.nx * 8
    return int(min(cfg.nt, max(32, budget // per_slice)))


def build_plan(stk, cfg, stream=None, time_chunk=0, transform="dst"):
    return stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, stream=stream, time_chunk=time_chunk,
                                   transform=transform)


def cpu_reference_run(cfg, steps: int, seed: int = 0):
    """The oracle port of solve_projected_heat_with on a causal prefix (steps slices),
    streamed in chunks with the modal recurrence carried; F generation is not timed."""
    from oracle import oracle as O
    from paper_1912_10082_b200 import inputs
    m, a = O.fem1d_matrices(0.0, 1.0, cfg.n)
    d, c = O.heat_time_matrices(cfg.nt)
    st = O.DecoupledStream([O.p1_pencil_eig(m, a)] * cfg.ndim, d, c)
    t = 0.0
    for j0 in range(0, steps, REF_MAX_CHUNK):
        F = inputs.heat_rhs_host_slices(cfg, j0, min(j0 + REF_MAX_CHUNK, steps), seed)
        t0 = time.perf_counter()
        st.step(F)
        t += time.perf_counter() - t0
    return t


def cpu_cn_run(cfg, steps: int = 16, seed: int = 0):
    """The reference's own CPU heat solver for a full-rank load: crank_nicolson
    (stk/cn_baseline.hpp:26-48; SimplicialLLT -> SuperLU), single thread as the reference
    runs it.  Times the factorisation plus `steps` steps; the full solve is
    extrapolated linearly in n_t (SPEC.md:523 records CN as linear in N_t)."""
    import scipy.sparse.linalg as spl
    from oracle import oracle as O
    from paper_1912_10082_b200 import inputs
    F = inputs.heat_rhs_host(cfg, seed, nsteps=steps)
    m, a = O.fem1d_matrices(0.0, 1.0, cfg.n)
    M, A = O.tensor_sparse([m] * cfg.ndim, [a] * cfg.ndim)
    dt = 1.0 / cfg.nt
    t0 = time.perf_counter()
    lu = spl.splu((M + (dt / 2.0) * A).tocsc())
    t_fac = time.perf_counter() - t0
    rhs = (M - (dt / 2.0) * A).tocsr()
    u = np.zeros(F.shape[1])
    t0 = time.perf_counter()
    for l in range(steps):
        u = lu.solve(rhs @ u + F[l])
    t_step = (time.perf_counter() - t0) / steps
    t_full = t_fac + cfg.nt * t_step
    return {"value": cfg.unknowns / t_full, "unit": UNIT, "cores": 1, "kind": "port",
            "factor_s": t_fac, "step_s": t_step, "full_solve_s_extrapolated": t_full,
            "sample": f"crank_nicolson (SuperLU, 1 thread): factorisation + {steps} of "
                      f"{cfg.nt} steps of {cfg.name}, extrapolated linearly in n_t"}


def binding_from_profiles():
    """The resource that actually bounds the half-length DST kernels (ncu, committed)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get("dst_half_binding_resource")
    except Exception:
        return None


def traffic_from_profiles(kind: str = "gemm"):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(f"{kind}_dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_reference(args):
    """The reference's CPU path on the SAME workload as the GPU arm: the oracle port of
    solve_projected_heat_with in tensor form (oracle.DecoupledStream, numpy + all-core BLAS)
    solving the full n_t time axis, split into args.steps consecutive chunks with the
    per-mode recurrence carried between them -- so the timed steps together are exactly one
    full solve of the configuration.  F is generated outside the timed region.  Only the
    host-only input generator of the package is imported; the product library is not mapped
    (the line lists what was)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1912_10082_b200 import inputs  # host-only module: does not load _stk_gpu.so
    cfg = inputs.CONFIGS[args.config]
    cores = os.cpu_count()
    m, a = O.fem1d_matrices(0.0, 1.0, cfg.n)
    d, c = O.heat_time_matrices(cfg.nt)
    eigs = [O.p1_pencil_eig(m, a)] * cfg.ndim
    warm = O.DecoupledStream(eigs, d, c)
    for w in range(args.warmup):  # warms BLAS threads and page-faults the work arrays
        warm.step(inputs.heat_rhs_host_slices(cfg, w, w + 1))
    steps = max(1, min(args.steps, cfg.nt))
    bounds = np.linspace(0, cfg.nt, steps + 1).astype(int)
    st = O.DecoupledStream(eigs, d, c)
    t_solve = 0.0
    t_wall0 = time.perf_counter()
    for k in range(steps):
        for j0 in range(bounds[k], bounds[k + 1], REF_MAX_CHUNK):
            j1 = min(j0 + REF_MAX_CHUNK, bounds[k + 1])
            F = inputs.heat_rhs_host_slices(cfg, j0, j1)
            t0 = time.perf_counter()
            st.step(F)
            t_solve += time.perf_counter() - t0
    wall = time.perf_counter() - t_wall0
    assert st.j == cfg.nt
    value = cfg.unknowns / t_solve
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "unknowns_per_step": cfg.unknowns / steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_solve / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"the full {args.config} solve (all {cfg.nt} time slices), "
                                   f"streamed as {steps} steps of consecutive time chunks "
                                   f"with the modal recurrence carried; oracle heat_decoupled "
                                   f"(numpy + {cores}-thread BLAS)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s_incl_input_generation": wall,
        "native_so_loaded": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)
    return 0


def line_binding_from_profiles():
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get("line_binding_resource")
    except Exception:
        return None


def fused_binding_from_profiles():
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get("fused_binding_resource")
    except Exception:
        return None


def _timed_path(stk, inputs, cfg, transform, args, stream, barrier, F, U, with_clocks):
    """Warm up and time args.steps solves of one transform backend on the plan stream (no
    profiling: 2D plans may run their overlapped multi-stream schedule), then one profiled
    pass of 2 solves (kernels back to back on the plan stream) for the per-kernel times."""
    import torch
    plan = build_plan(stk, cfg, stream=stream.cuda_stream, transform=transform)
    for _ in range(args.warmup):
        plan.solve(F, out=U)
    stream.synchronize()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) if with_clocks else None
    if clocks:
        clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.solve(F, out=U)
    e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1)
    nprof = 2
    plan.profile_begin()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(nprof):
        plan.solve(F, out=U)
    p1.record(stream)
    stream.synchronize()
    prof = plan.profile_end()
    ms_seq = p0.elapsed_time(p1) / nprof  # the same solve with its kernels back to back
    relres, _ = plan.residual(U, F)
    t_ms, t_n = prof["transform"]
    s_ms, s_n = prof["scan"]
    N = cfg.unknowns
    sec = ms / 1e3 / args.steps
    sched = plan.schedule() if transform == "dst" else "separate"
    fused = sched != "separate"
    line = sched == "line_solve"
    if transform == "dense":
        flops = 2.0 * cfg.n * N  # 2n flop per unknown per axis transform launch
        achieved = flops / (t_ms / t_n / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "gemm_f64_kernel (DMMA basis transforms)",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic_from_profiles(),
                "peak_source": FP64_PEAK_SOURCE,
                "whole_solve_frac": (2 * cfg.ndim * flops * args.steps / (ms / 1e3) / 1e12)
                / FP64_PEAK_TFLOPS}
        roof["share_of_step"] = t_ms / nprof / (ms_seq)
    else:
        half = half_kernels(cfg)
        fft_flops = fft_flop_per_unknown(cfg.n, half)  # per element and axis pass
        t_hbm = 16.0 * N / (HBM_GBS * 1e9)  # read F + write U once
        rec_flops = 12.0  # recurrence: 2 FMA pivot/coupling, Newton reciprocal, update, weight
        # line-solve schedule: axis 0 is not transformed; per unknown 4 ops for the right-hand
        # side, 2 + 1 + 4 for the zero-start / causal / anti-causal sweeps (FMA = 2 flop)
        line_flops = 20.0
        exec_flops = (2 * (cfg.ndim - 1) * fft_flops + line_flops) if line else \
            (2 * cfg.ndim * fft_flops + rec_flops)
        t_fp64 = exec_flops * N / (FP64_PEAK_TFLOPS * 1e12)
        passes = (t_n + s_n) / nprof  # HBM passes of the executed schedule per solve
        t_tr = t_ms / t_n  # mean transform-only pass
        contig = {"kernel": "dst_half_kernel (contiguous axis, forward / inverse)",
                  "ms_per_launch": t_tr, "achieved_gbs": 16.0 * N / (t_tr / 1e3) / 1e9,
                  "frac_hbm": 16.0 * N / (t_tr / 1e3) / 1e9 / HBM_GBS,
                  "launches_per_solve": t_n / nprof}
        if line:
            # the contiguous transform passes are the larger share of the step; the line pass
            # (class 1 of the profile) is reported beside them
            t_f = s_ms / s_n
            achieved = 16.0 * N / (t_tr / 1e3) / 1e9
            roof = {"bound": "hbm",
                    "kernel": "dst_half_bulk_kernel / dst_half_kernel (FP64 half-length DST-I along "
                              "the contiguous axis, forward and inverse: N-point Stockham FFT per "
                              "vector pair; N = 1024 takes each pair by one bulk copy)",
                    "achieved": achieved, "peak": HBM_GBS, "unit": "GB/s",
                    "frac": achieved / HBM_GBS,
                    "traffic": traffic_from_profiles("dst_half"),
                    "binding_resource": binding_from_profiles(),
                    "ms_per_launch": t_tr, "launches_per_solve": t_n / nprof,
                    "share_of_sequential_step": t_ms / nprof / ms_seq,
                    "other_kernel": {
                        "kernel": "heat_tridiag_tma_kernel (time-marching line solves along "
                                  "axis 0: constant-coefficient causal / anti-causal sweeps, TMA "
                                  "tile loads and stores; one read + one write of S)",
                        "ms_per_launch": t_f, "achieved_gbs": 16.0 * N / (t_f / 1e3) / 1e9,
                        "frac_hbm": 16.0 * N / (t_f / 1e3) / 1e9 / HBM_GBS,
                        "flop_per_unknown": line_flops,
                        "traffic": traffic_from_profiles("line"),
                        "binding_resource": line_binding_from_profiles(),
                        "launches_per_solve": s_n / nprof,
                        "share_of_sequential_step": s_ms / nprof / ms_seq}}
        elif fused:
            t_f = s_ms / s_n
            achieved = 16.0 * N / (t_f / 1e3) / 1e9
            roof = {"bound": "hbm",
                    "kernel": "heat_fused_axis0_kernel (time-marching: forward DST-I along axis 0, "
                              "modal recurrence, inverse DST-I; one read + one write of S)",
                    "achieved": achieved, "peak": HBM_GBS, "unit": "GB/s",
                    "frac": achieved / HBM_GBS,
                    "traffic": traffic_from_profiles("fused"),
                    "binding_resource": fused_binding_from_profiles(),
                    "ms_per_launch": t_f,
                    "flop_per_unknown": 2 * fft_flops + rec_flops,
                    "fp64_tflops": (2 * fft_flops + rec_flops) * N / (t_f / 1e3) / 1e12,
                    "share_of_sequential_step": s_ms / nprof / ms_seq,
                    "other_kernel": contig}
        else:
            achieved = 16.0 * N / (t_tr / 1e3) / 1e9
            kname = ("dst_half_kernel / dst_half_strided2_kernel (FP64 half-length DST-I: "
                     "N-point Stockham FFT per vector pair)") if half else \
                "dst_axis_kernel / dst_strided_kernel (FP64 padded 2N-point FFT DST-I)"
            roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": HBM_GBS,
                    "unit": "GB/s", "frac": achieved / HBM_GBS,
                    "traffic": traffic_from_profiles("dst_half" if half else "dst"),
                    "binding_resource": binding_from_profiles() if half else None,
                    "share_of_sequential_step": t_ms / nprof / ms_seq}
        roof.update({
            "peak_source": HBM_SOURCE,
            "flop_per_unknown_per_transform_pass": fft_flops,
            "whole_solve_frac": max(t_hbm, t_fp64) / sec,
            "whole_solve_basis": "SURVEY 8(d): T_roof = max(16 B/unknown / HBM, executed "
                                 "DST + recurrence flops / FP64 peak) over the measured solve",
            "whole_solve_roof_ms": 1e3 * max(t_hbm, t_fp64),
            "hbm_passes_per_solve": passes,
            "whole_solve_frac_executed_passes": passes * t_hbm / sec,
            "sequential_ms_per_step": ms_seq,
            "overlap_gain_ms": ms_seq - 1e3 * sec})
    out = {"transform": transform, "ms_per_step": ms / args.steps, "ms": ms,
           "value": N * args.steps / (ms / 1e3), "relres_gpu_k1": relres, "roofline": roof,
           "launches": int(round((t_n + s_n) / nprof * args.steps)),
           "schedule": sched,
           "recurrence_kernel": {"kernel": {"line_solve": "heat_tridiag_tma_kernel",
                                            "fused_dst": "heat_fused_axis0_kernel",
                                            "separate": "heat_scan_kernel"}[sched],
                                 "ms_per_launch": s_ms / s_n,
                                 "gbs": 16.0 * N / (s_ms / s_n / 1e3) / 1e9,
                                 "frac_hbm": 16.0 * N / (s_ms / s_n / 1e3) / 1e9 / HBM_GBS}}
    return plan, out, clk


def heat_config_leg(stk, inputs, name, stream, steps=10, warmup=3, with_cpu=True,
                    cpu_slices=None):
    """One named heat shape: the device solve with dense F resident in
    HBM (P1_DST backend, CUDA events on the plan stream), the factored-load solve of the same
    low-rank F, the GPU K1 relres, the whole-solve roofline fraction (T_roof = max(16
    B/unknown / HBM, executed flops / FP64) over the measured time), and the oracle port of
    the reference's CPU path on this host (full n_t, or a causal prefix when stated)."""
    import torch
    cfg = inputs.CONFIGS[name]
    N = cfg.unknowns
    with torch.cuda.stream(stream):
        plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst",
                                       stream=stream.cuda_stream)
        F = inputs.heat_rhs_device(cfg)
        U = torch.empty_like(F)
        for _ in range(warmup):
            plan.solve(F, out=U)
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            plan.solve(F, out=U)
        e1.record(stream)
        stream.synchronize()
        ms = e0.elapsed_time(e1) / steps
        plan.profile_begin()
        plan.solve(F, out=U)
        prof = plan.profile_end()
        relres, _ = plan.residual(U, F)
        out = {"workload": cfg.name, "unknowns": N, "ms": ms, "value": N / (ms / 1e3),
               "relres_gpu_k1": relres,
               "launches_per_solve": prof["transform"][1] + prof["scan"][1]}
        half = half_kernels(cfg)
        sched = plan.schedule()
        out["schedule"] = sched
        fft = fft_flop_per_unknown(cfg.n, half)
        fl = ((2 * (cfg.ndim - 1) * fft + 20.0) if sched == "line_solve"
              else (2 * cfg.ndim * fft + 12.0)) * N
        t_roof = max(16.0 * N / (HBM_GBS * 1e9), fl / (FP64_PEAK_TFLOPS * 1e12))
        out["roofline"] = {"bound": "hbm" if 16.0 * N / HBM_GBS / 1e9 >= fl / FP64_PEAK_TFLOPS
                           / 1e12 else "fp64", "roof_ms": 1e3 * t_roof,
                           "frac": t_roof / (ms / 1e3), "flops_executed": fl,
                           "bytes_alg": 16.0 * N}
        if cfg.rank:
            left, right = inputs.heat_factors(cfg)
            L = torch.tensor(left.T.copy(), device="cuda")
            R = torch.tensor(right.T.copy(), device="cuda")
            for _ in range(warmup):
                plan.solve_factored(L, R, out=U)
            e0.record(stream)
            for _ in range(steps):
                plan.solve_factored(L, R, out=U)
            e1.record(stream)
            stream.synchronize()
            msf = e0.elapsed_time(e1) / steps
            out["factored"] = {"ms": msf, "value": N / (msf / 1e3),
                               "bytes_alg": 8.0 * N,
                               "frac_hbm": 8.0 * N / (HBM_GBS * 1e9) / (msf / 1e3)}
        plan.close()
        del F, U
    if with_cpu:
        from oracle import oracle as O
        m, a = O.fem1d_matrices(0.0, 1.0, cfg.n)
        d, c = O.heat_time_matrices(cfg.nt)
        st = O.DecoupledStream([O.p1_pencil_eig(m, a)] * cfg.ndim, d, c)
        nts = cfg.nt if cpu_slices is None else cpu_slices
        tc = 0.0
        for j0 in range(0, nts, REF_MAX_CHUNK):
            j1 = min(j0 + REF_MAX_CHUNK, nts)
            Fh = inputs.heat_rhs_host_slices(cfg, j0, j1)
            t0 = time.perf_counter()
            st.step(Fh)
            tc += time.perf_counter() - t0
        vc = cfg.nx * nts / tc
        out["cpu_baseline"] = {"value": vc, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                               "s": tc, "sample": (f"full solve ({nts} slices)" if nts == cfg.nt
                                                   else f"causal prefix of {nts} of {cfg.nt} "
                                                        "slices") +
                               ", oracle heat_decoupled (numpy + all-core BLAS)"}
        out["gpu_over_cpu"] = out["value"] / vc
    return out


def rksm_leg(stk, inputs, with_cpu=True, name="cfg1"):
    """the paper's rational Krylov solver (rksm_solve, stk/rksm.hpp:127-234)
    on the BASELINE rank-1 config, next to the direct decoupled solve of the same factored
    load.  Wall-clock around the synchronous C-ABI call (it interleaves host decisions)."""
    import torch
    cfg = inputs.CONFIGS[name]
    left, right = inputs.heat_factors(cfg)
    L = torch.tensor(left.T.copy(), device="cuda")
    R = torch.tensor(right.T.copy(), device="cuda")
    plan = stk.HeatPlan.p1_uniform(cfg.ndim, cfg.n, cfg.nt, transform="dst")
    plan.rksm(L, R, tol=1e-8, maxit=100)  # warm-up: grows every scratch / pinned buffer
    reps = 5
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        _, _, rep = plan.rksm(L, R, tol=1e-8, maxit=100)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / reps
    plan.solve_factored(L, R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        plan.solve_factored(L, R)
    torch.cuda.synchronize()
    td = (time.perf_counter() - t0) / reps
    out = {"workload": cfg.name, "tol": 1e-8, "iterations": rep.iterations,
           "final_relres": rep.final_relres, "converged": rep.converged, "rank": rep.rank,
           "mu_mem": rep.mu_mem, "ms": 1e3 * t, "unknowns_per_s": cfg.unknowns / t,
           "direct_ms": 1e3 * td, "direct_unknowns_per_s": cfg.unknowns / td}
    if with_cpu:
        sys.path.insert(0, str(ROOT))
        from oracle import oracle as orc
        m, a = orc.fem1d_matrices(0.0, 1.0, cfg.n)
        d, c = orc.heat_time_matrices(cfg.nt)
        t0 = time.perf_counter()
        _, _, its, _ = orc.rksm_solve([m], [a], d, c, left, right, tol=1e-8, maxit=100)
        out["cpu_oracle"] = {"s": time.perf_counter() - t0, "iterations": its, "cores": 1,
                             "kind": "port (numpy/scipy SuperLU restatement)"}
    plan.close()
    return out


def _event_ms(stream, fn, reps):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) / reps


def wave_leg(stk, inputs, with_cpu=True, cpu_iters=10):
    """SURVEY 8(a) rows a8-a10 on BASELINE config 4 (1D wave, cubic splines, 1023 x 1025).
    Headline: PCG with the space-modal time-banded preconditioner (stkg_modal_banded_solve)
    to 1e-7, and the double-double refined solve to the north_star 1e-10 bar.  Beside it the
    reference's preconditioner (TwoTermPrecond): PCG to 1e-7 and the reference's GMRES for a
    fixed 300-iteration budget.  The reference-faithful oracle GMRES (numpy + multithreaded
    BLAS) is timed per iteration on the host for a bounded number of iterations."""
    import torch
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    plan = stk.WavePlan(sm, tm, preconditioner="modal_banded")
    Fh = inputs.wave_rhs_host(cfg)
    F = torch.tensor(Fh, device="cuda")
    N = cfg.nh * (cfg.nt + 1)
    stream = torch.cuda.current_stream()
    # --- headline: modal banded preconditioner
    plan.pcg(F, tol=1e-7, maxit=500)  # warm-up (sizes the Krylov workspace)
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        _, rm = plan.pcg(F, tol=1e-7, maxit=500)
    torch.cuda.synchronize()
    tm_ = (time.perf_counter() - t0) / reps
    plan.solve_refined(F, tol=1e-10, inner_tol=1e-6, max_refine=6)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        _, _, rr = plan.solve_refined(F, tol=1e-10, inner_tol=1e-6, max_refine=6)
    torch.cuda.synchronize()
    tr = (time.perf_counter() - t0) / reps
    w = torch.empty_like(F)
    y = torch.empty_like(F)
    ms_prec = _event_ms(stream, lambda: plan.modal_banded_solve(F, out=w), 20)
    ms_tt = _event_ms(stream, lambda: plan.two_term_solve(F, out=w), 20)
    ms_op = _event_ms(stream, lambda: plan.apply(F, out=y), 20)
    # 2 GEMMs of 2 nh^2 nt flop + 2 banded triangular solves (~14 flop/unknown) + operator
    fl_prec = 2 * 2.0 * cfg.nh * cfg.nh * (cfg.nt + 1) + 14.0 * N
    fl_iter = fl_prec + 84.0 * N
    out = {"workload": cfg.name, "unknowns": N,
           "pcg": {"preconditioner": "modal_banded", "iterations": rm.iterations,
                   "final_relres": rm.final_relres, "tol": 1e-7, "s": tm_,
                   "ms_per_iteration": 1e3 * tm_ / max(rm.iterations, 1),
                   "unknowns_per_s": N / tm_,
                   "roofline": {"bound": "tensor", "flop_per_iteration": fl_iter,
                                "roof_ms_per_iteration": 1e3 * fl_iter / (FP64_PEAK_TFLOPS * 1e12),
                                "peak": FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
                                "frac": (1e3 * fl_iter / (FP64_PEAK_TFLOPS * 1e12))
                                / (1e3 * tm_ / max(rm.iterations, 1)),
                                "basis": "2 DMMA GEMMs + 2 banded solves per spatial mode "
                                         "(stkg_modal_banded_solve) + the banded WaveOperator "
                                         "per iteration; wall clock incl. the host "
                                         "convergence checks"}},
           "refined_dd": {"tol": 1e-10, "rounds": len(rr.rel_res_history) - 1,
                          "pcg_iterations": rr.iterations, "final_relres_dd": rr.final_relres,
                          "history": rr.rel_res_history, "converged": rr.converged, "s": tr,
                          "unknowns_per_s": N / tr,
                          "note": "mixed-precision iterative refinement, residual in "
                                  "double-double (stkg_wave_solve_refined), modal banded "
                                  "preconditioner"},
           "kernels_ms": {"modal_banded_solve": ms_prec, "two_term_solve": ms_tt,
                          "wave_apply": ms_op,
                          "modal_banded_tflops": fl_prec / (ms_prec / 1e3) / 1e12}}
    # --- the reference's preconditioner (TwoTermPrecond)
    plan.set_preconditioner("two_term")
    plan.gmres(F, stk.GmresConfig(tol=0.999, maxit=300))  # sizes the 301-column basis
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rg = plan.gmres(F, stk.GmresConfig(tol=1e-9, maxit=300))
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rp = plan.pcg(F, tol=1e-7, maxit=6000)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    fl = WAVE_FLOP_PER_PCG_ITER(cfg.nh, cfg.nt + 1)
    roof_ms = 1e3 * fl / (FP64_PEAK_TFLOPS * 1e12)
    out["two_term"] = {
        "gmres": {"iterations": rg.iterations, "final_relres": rg.final_relres,
                  "s": tg, "ms_per_iteration": 1e3 * tg / max(rg.iterations, 1)},
        "pcg": {"iterations": rp.iterations, "final_relres": rp.final_relres, "tol": 1e-7,
                "s": tp, "ms_per_iteration": 1e3 * tp / max(rp.iterations, 1),
                "unknowns_per_s": N / tp,
                "roofline": {"bound": "tensor", "flop_per_iteration": fl,
                             "roof_ms_per_iteration": roof_ms,
                             "frac": roof_ms / (1e3 * tp / max(rp.iterations, 1)),
                             "basis": "4 DMMA GEMMs of TwoTermPrecond::solve + the banded "
                                      "WaveOperator per iteration"}}}
    if with_cpu:
        sys.path.insert(0, str(ROOT))
        from oracle import oracle as orc
        sb = np.stack([sm.M.band, sm.A.band, sm.Q.band])
        tb = np.stack([tm.Q.band, tm.D.band, tm.M.band])
        ws = orc.WaveSystemNP(sb, tb)
        b = np.ascontiguousarray(Fh).ravel()
        t0 = time.perf_counter()
        _, its, _ = ws.gmres(b, tol=1e-14, maxit=cpu_iters)
        tc = time.perf_counter() - t0
        out["cpu_oracle_gmres"] = {"iterations": its, "s": tc,
                                   "ms_per_iteration": 1e3 * tc / max(its, 1),
                                   "cores": os.cpu_count(), "kind": "port",
                                   "sample": f"{its} reference-faithful GMRES iterations "
                                             "(numpy/scipy, MGS + re-orth, dense eigenbasis "
                                             "TwoTermPrecond) on the full config-4 system"}
    plan.close()
    return out


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1912_10082_b200 as stk
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    stream = torch.cuda.Stream()
    N = cfg.unknowns

    def barrier():
        if dist is not None:
            dist.barrier()

    main = args.transform
    alt = "dense" if main == "dst" else "dst"
    with torch.cuda.stream(stream):
        F = inputs.heat_rhs_device(cfg, seed=rank)
        U = torch.empty_like(F)
        stream.synchronize()
        plan, res, clk = _timed_path(stk, inputs, cfg, main, args, stream, barrier, F, U, True)
        # K1 residual kernel (not part of the solve): HBM roofline, 16 B/unknown
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        plan.residual(U, F)
        r1.record(stream)
        stream.synchronize()
        k1_ms = r0.elapsed_time(r1)
        plan.close()
        alt_res = None
        if not args.no_alt:
            aplan, alt_res, _ = _timed_path(stk, inputs, cfg, alt, args, stream, barrier, F, U,
                                            False)
            aplan.close()
    ms_max = max_over_ranks(res["ms"], dist, "cuda")
    value = aggregate_value(N, args.steps, world, ms_max)

    # ---- end to end through the public host-buffer API --------------------------------
    e2e = None
    if not args.no_e2e:
        import dataclasses
        ne = e2e_slices(cfg, world)
        cfg_e = cfg if ne == cfg.nt else dataclasses.replace(cfg, nt=ne)
        N_e = cfg_e.nx * cfg_e.nt
        Fh = torch.empty((cfg_e.nt, cfg_e.nx), dtype=torch.float64).pin_memory()
        Uh = torch.empty_like(Fh).pin_memory()
        Fh.copy_(F[:ne])
        del U
        torch.cuda.empty_cache()
        plan_h = build_plan(stk, cfg_e, stream=stream.cuda_stream, time_chunk=args.time_chunk,
                            transform=main)
        plan_h.solve_host(Fh.numpy(), out=Uh.numpy())  # warm-up (allocates chunk buffers)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan_h.solve_host(Fh.numpy(), out=Uh.numpy())
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        t_e = max_over_ranks(t_e2e, dist, "cuda")
        e2e = {"value": aggregate_value(N_e, args.e2e_steps, world, 1e3 * t_e), "unit": UNIT,
               "h2d_bytes_per_step": N_e * 8, "d2h_bytes_per_step": N_e * 8,
               "steps": args.e2e_steps, "time_slices": ne,
               "api": "stkg_heat_solve_host (pinned host buffers)"}
        plan_h.close()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg),
        "backend": {"transform": main, "parallelism": "replicas" if world > 1 else "single"},
        "relres_gpu_k1": res["relres_gpu_k1"],
        "roofline": res["roofline"],
        "e2e": e2e,
        "gpu_launches": res["launches"],
        "schedule": res.get("schedule"),
        "k1_residual": {"ms": k1_ms, "gbs": 16.0 * N / (k1_ms / 1e3) / 1e9,
                        "frac_hbm": 16.0 * N / (k1_ms / 1e3) / 1e9 / HBM_GBS,
                        "bytes_alg": 16 * N},
        "recurrence_kernel": res["recurrence_kernel"],
        "clocks": clk,
    }
    if args.config == "cfg3":
        # >= 60% of the dense-transform roofline = <= 365 ms per solve
        line["north_star_target"] = {
            "bar_ms_per_step": 365.0, "bar_unknowns_per_s": 2.93e9,
            "value_over_bar": value / 2.93e9,
            "note": "BASELINE.md target for cfg3 (>= 60% of the dense DMMA-transform roofline "
                    "at 40 TF); the executed algorithm (fast sine transforms) has its own, "
                    "lower roofline -- see roofline / DESIGN.md K2b"}
    if alt_res is not None:
        line["alt_path"] = alt_res
    if rank == 0 and not args.no_rksm:
        line["rksm"] = rksm_leg(stk, inputs, with_cpu=(world == 1 and not args.no_cpu))
    if rank == 0 and not args.no_wave:
        line["wave"] = wave_leg(stk, inputs, with_cpu=(world == 1 and not args.no_cpu))
    if rank == 0 and not args.no_configs:
        cfgs = {}
        for nm, slices in (("cfg1", None), ("cfg2", None), ("cfg5", 32)):
            cfgs[nm] = heat_config_leg(stk, inputs, nm, stream,
                                       with_cpu=(world == 1 and not args.no_cpu),
                                       cpu_slices=slices)
        cfgs[args.config] = {"workload": cfg.name, "unknowns": N, "ms": ms_max / args.steps,
                             "value": value / world, "relres_gpu_k1": res["relres_gpu_k1"],
                             "roofline": {"frac": res["roofline"].get("whole_solve_frac"),
                                          "roof_ms": res["roofline"].get("whole_solve_roof_ms"),
                                          "note": "the headline line (roofline.whole_solve_*)"}}
        if "wave" in line:
            wv = line["wave"]
            cfgs["cfg4"] = {"workload": wv["workload"], "unknowns": wv["unknowns"],
                            "solve_s_1e-7": wv["pcg"]["s"],
                            "value": wv["pcg"]["unknowns_per_s"],
                            "pcg_ms_per_iteration": wv["pcg"]["ms_per_iteration"],
                            "pcg_iterations_1e-7": wv["pcg"]["iterations"],
                            "roofline": wv["pcg"]["roofline"],
                            "refined_dd_relres": wv["refined_dd"]["final_relres_dd"],
                            "refined_s": wv["refined_dd"]["s"],
                            "two_term_pcg_iterations_1e-7": wv["two_term"]["pcg"]["iterations"],
                            "two_term_pcg_s": wv["two_term"]["pcg"]["s"],
                            "cpu_baseline": wv.get("cpu_oracle_gmres")}
        line["configs"] = dict(sorted(cfgs.items()))
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_t = cpu_reference_run(cfg, args.ref_sample)
        cpu_v = cfg.nx * args.ref_sample / cpu_t
        if not args.no_cn:
            line["cpu_reference_cn"] = cpu_cn_run(cfg)
        line["cpu_baseline"] = {"value": cpu_v, "unit": UNIT, "cores": os.cpu_count(),
                                "kind": "port",
                                "sample": f"oracle heat_decoupled (numpy+BLAS), "
                                          f"{args.ref_sample}-slice causal prefix of {args.config}, "
                                          f"{cpu_t:.2f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg5"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--time-chunk", type=int, default=0)
    ap.add_argument("--ref-sample", type=int, default=CPU_SAMPLE_STEPS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rksm", action="store_true", help="skip the RKSM (cfg1) side leg")
    ap.add_argument("--no-wave", action="store_true", help="skip the wave (cfg4) side leg")
    ap.add_argument("--no-cn", action="store_true",
                    help="skip the single-thread Crank-Nicolson CPU reference timing")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other transform backend")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config legs (cfg1, cfg2, cfg5 heat; cfg4 from the wave leg)")
    ap.add_argument("--transform", choices=["dst", "dense"], default="dst",
                    help="headline backend: P1 fast sine transforms (dst) or dense DMMA GEMMs")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
