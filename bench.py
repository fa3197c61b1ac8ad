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
HBM_GBS = 6557.4  # MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)
CPU_SAMPLE_STEPS = 96  # causal prefix of cfg3 time slices for the CPU leg


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
    """The oracle port of solve_projected_heat_with on a causal prefix (steps slices)."""
    from oracle import oracle as O
    from paper_1912_10082_b200 import inputs
    F = inputs.heat_rhs_host(cfg, seed, nsteps=steps)
    m, a = O.fem1d_matrices(0.0, 1.0, cfg.n)
    d, c = O.heat_time_matrices(cfg.nt)
    eig = O.p1_pencil_eig(m, a)
    t0 = time.perf_counter()
    O.heat_decoupled([eig] * cfg.ndim, d, c, F, nsteps=steps)
    return time.perf_counter() - t0


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
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1912_10082_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    cores = os.cpu_count()
    steps_per = args.ref_sample
    for _ in range(args.warmup):
        cpu_reference_run(cfg, max(2, steps_per // 8))
    times = [cpu_reference_run(cfg, steps_per) for _ in range(args.steps)]
    t = sum(times)
    value = cfg.nx * steps_per * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "parallelism": "cpu",
                   "sample": f"causal prefix of {steps_per} of {cfg.nt} time slices"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"oracle heat_decoupled (numpy+BLAS, {cores} threads), "
                                   f"{steps_per}-slice causal prefix of {args.config}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _timed_path(stk, inputs, cfg, transform, args, stream, barrier, F, U, with_clocks):
    """Warm up and time args.steps solves of one transform backend on the plan stream."""
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
    plan.profile_begin()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.solve(F, out=U)
    e1.record(stream)
    stream.synchronize()
    prof = plan.profile_end()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1)
    relres, _ = plan.residual(U, F)
    t_ms, t_n = prof["transform"]
    s_ms, s_n = prof["scan"]
    N = cfg.unknowns
    if transform == "dense":
        flops = 2.0 * cfg.n * N  # 2n flop per unknown per axis transform launch
        achieved = flops / (t_ms / t_n / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "gemm_f64_kernel (DMMA basis transforms)",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic_from_profiles(),
                "peak_source": FP64_PEAK_SOURCE,
                "whole_solve_frac": (2 * cfg.ndim * flops * args.steps / (ms / 1e3) / 1e12)
                / FP64_PEAK_TFLOPS}
    else:
        bytes_launch = 16.0 * N  # read + write each unknown once per axis pass
        achieved = bytes_launch / (t_ms / t_n / 1e3) / 1e9
        # which sine-transform kernels the plan runs (heat.cu::dst_pass)
        half = (cfg.ndim >= 2 and cfg.n + 1 in (512, 1024)
                and os.environ.get("STKG_DST_HALF", "1") != "0")
        L = (cfg.n + 1) if half else 2 * (cfg.n + 1)  # complex FFT length per vector pair
        fft_flops = 5.0 * L * np.log2(L) / 2.0 / cfg.n  # per element and axis pass
        kname = ("dst_half_kernel / dst_half_strided2_kernel (FP64 half-length DST-I: "
                 "N-point Stockham FFT per vector pair)") if half else \
            "dst_axis_kernel / dst_strided_kernel (FP64 padded 2N-point FFT DST-I)"
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": achieved, "peak": HBM_GBS, "unit": "GB/s",
                "frac": achieved / HBM_GBS,
                "traffic": traffic_from_profiles("dst_half" if half else "dst"),
                "binding_resource": binding_from_profiles() if half else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "flop_per_unknown_per_pass": fft_flops,
                "whole_solve_frac": ((2 * cfg.ndim + 1) * 16.0 * N * args.steps / (ms / 1e3) / 1e9)
                / HBM_GBS}
    roof["share_of_step"] = t_ms / ms
    roof["scan_share_of_step"] = s_ms / ms
    out = {"transform": transform, "ms_per_step": ms / args.steps, "ms": ms,
           "value": N * args.steps / (ms / 1e3), "relres_gpu_k1": relres, "roofline": roof,
           "launches": int(t_n + s_n),
           "k3_scan": {"ms_per_launch": s_ms / s_n, "gbs": 16.0 * N / (s_ms / s_n / 1e3) / 1e9,
                       "frac_hbm": 16.0 * N / (s_ms / s_n / 1e3) / 1e9 / HBM_GBS}}
    return plan, out, clk


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


def wave_leg(stk, inputs, with_cpu=True, cpu_iters=10):
    """SURVEY 8(a) rows a8-a10 on BASELINE config 4 (1D wave, cubic splines, 1023 x 1025):
    the reference's GMRES + TwoTermPrecond for a fixed 300-iteration budget and the PCG
    performance path, timed on the device; the reference-faithful oracle GMRES (numpy +
    multithreaded BLAS) timed per iteration on the host for a bounded number of iterations."""
    import torch
    cfg = inputs.CONFIGS["cfg4"]
    sm = stk.wave_space_matrices(stk.SpaceGrid1D(0.0, 1.0, cfg.nh))
    tm = stk.wave_time_matrices(stk.TimeGrid(cfg.nt, 1.0))
    plan = stk.WavePlan(sm, tm)
    Fh = inputs.wave_rhs_host(cfg)
    F = torch.tensor(Fh, device="cuda")
    # warm-up: sizes the 301-column Krylov basis (gmres_run reserves maxit + 1 columns up
    # front) and exits after the first iteration, so no allocation lands in the timed run
    plan.gmres(F, stk.GmresConfig(tol=0.999, maxit=300))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rg = plan.gmres(F, stk.GmresConfig(tol=1e-9, maxit=300))
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, rp = plan.pcg(F, tol=1e-7, maxit=6000)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, _, rr = plan.solve_refined(F, tol=1e-10, inner_tol=1e-6, max_refine=6)
    torch.cuda.synchronize()
    tr = time.perf_counter() - t0
    N = cfg.nh * (cfg.nt + 1)
    out = {"workload": cfg.name, "unknowns": N,
           "refined_dd": {"tol": 1e-10, "rounds": len(rr.rel_res_history) - 1,
                          "pcg_iterations": rr.iterations, "final_relres_dd": rr.final_relres,
                          "history": rr.rel_res_history, "converged": rr.converged, "s": tr,
                          "note": "mixed-precision iterative refinement, residual in "
                                  "double-double (stkg_wave_solve_refined)"},
           "gmres": {"iterations": rg.iterations, "final_relres": rg.final_relres,
                     "s": tg, "ms_per_iteration": 1e3 * tg / max(rg.iterations, 1)},
           "pcg": {"iterations": rp.iterations, "final_relres": rp.final_relres, "tol": 1e-7,
                   "s": tp, "ms_per_iteration": 1e3 * tp / max(rp.iterations, 1),
                   "unknowns_per_s": N / tp}}
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
                                             "preconditioner) on the full config-4 system"}
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
        "config": {"workload": cfg.name, "unknowns_per_step": N, "n": cfg.n, "nt": cfg.nt,
                   "transform": main,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2_flush": "inputs larger than L2 (F, U 8.6 GB each)",
                   "relres_gpu_k1": res["relres_gpu_k1"]},
        "roofline": res["roofline"],
        "e2e": e2e,
        "gpu_launches": res["launches"],
        "k1_residual": {"ms": k1_ms, "gbs": 16.0 * N / (k1_ms / 1e3) / 1e9,
                        "frac_hbm": 16.0 * N / (k1_ms / 1e3) / 1e9 / HBM_GBS,
                        "bytes_alg": 16 * N},
        "k3_scan": res["k3_scan"],
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
