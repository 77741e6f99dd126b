#!/usr/bin/env python
"""Benchmark of the parareal fine-propagator sweep (BASELINE.json metric).

One *step* is one fine sweep (``fine_sweep_intervals``, stepping.py:189-243)
over every slice a GPU owns, with the coarse states already resident in HBM.
Default workload: BASELINE config 3 (1-D sine Galerkin, M=512, P=64 slices,
m=1024 fine steps per slice, alpha=0.3, T=2) — the largest 1-D config and the
first on which a roofline binds; config 2 (``configs[1]``) is
latency-bound with 16 slices and is a parity case.  ``--config`` selects 1-5
(config 5: the BASELINE problem, P = 512 slices, at one GPU; 64 per GPU above).

    python bench.py [--gpus N --steps K --warmup W --config 3]
    python bench.py --impl reference ...      # CPU arm: the oracle port (+ the unmodified
                                              # reference on the Chebyshev form) on the host cores

With N > 1 (under torchrun, or ``--gpus N`` alone, which spawns N NCCL
ranks) each rank sweeps its contiguous block of a global problem with P*N
slices (parareal._block_bounds, parareal.py:62-72): weak scaling, no
collective inside the sweep.  Timing: CUDA events on the launch
stream, barrier + synchronize on both sides, max over ranks; the history
paths (P x (m+1) x M fp64 = 269 MB at config 3) exceed the 126 MB L2, so no
explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1  # measured DMMA/DFMA on this pool (profiles/fp64_peaks_r01.txt)


def _peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except OSError:
        pass
    return p


# --------------------------------------------------------------------------
# clocks sampler (NVML) during the timed region
# --------------------------------------------------------------------------
_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in _REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# algorithmic work of one fine-sweep launch
# --------------------------------------------------------------------------
def sweep_flops(M, m, slices, n_lo, pcg_iterations, solves):
    """Flops the matrix-free sine sweep does per launch, from its own counters.

    per substep:   (2 + 2 n_it) FFTs of length Q=2M at 5 Q log2 Q,
                   history 2 (r+1) M (blocked Toeplitz GEMM + near rows),
                   bracket 2 n M, PCG vector work 12 M per iteration,
                   pointwise/pre/post 30 Q.
    """
    Q = 2 * M
    fft = 5.0 * Q * math.log2(Q)
    units = slices * m
    it = pcg_iterations
    f = (2 * units + 2 * it) * fft
    f += slices * (m * (m + 1) + m) * M          # sum_r 2 (r) M  (r = 1..m) incl. b_{r-1} c_0
    f += sum(2.0 * n * M * m for n in range(n_lo, n_lo + slices))
    f += 12.0 * M * it + 30.0 * Q * units
    return f


def sweep_flops_2d(M, m, slices, n_lo, pcg_iterations):
    """2-D sweep work per launch: setup = 4M + 4Q line FFTs, each PCG iteration
    2M + 2Q line FFTs (length Q, 5 Q log2 Q), history 2 (r+1) M^2, bracket 2 n M^2,
    pointwise 40 Q^2 per setup and 6 Q^2 per iteration."""
    Q = 2 * M
    fft = 5.0 * Q * math.log2(Q)
    units = slices * m
    it = pcg_iterations
    f = units * (4 * M + 4 * Q) * fft + it * (2 * M + 2 * Q) * fft
    f += slices * (m * (m + 1) + m) * M * M
    f += sum(2.0 * n * M * M * m for n in range(n_lo, n_lo + slices))
    f += 40.0 * Q * Q * units + 6.0 * Q * Q * it
    return f


def history_bytes(M, m, slices, hb=8, group=1):
    """Bytes of the blocked history: each path row read once per block + written once.
    group = G > 1 (the TMA-fed DMMA helper, pf_kernels.cuh TC_G): the rows older than G + 1
    blocks are read once per super-block of G blocks, the (G + t) hb newest rows once per tile."""
    if group <= 1:
        rows_read = sum(((r0 + 1)) for r0 in range(0, m, hb))
    else:
        nblocks = (m + hb - 1) // hb
        rows_read = 0
        for beta in range(nblocks):
            S, t = divmod(beta, group)
            far = max(beta - 1, 0) * hb
            common = max(group * S - group - 1, 0) * hb
            rows_read += far - common                       # appended per tile
            if t == 0 and group * (S + 1) < nblocks:
                rows_read += max(group * S - 1, 0) * hb     # next super-block's common pass
    return slices * 8.0 * M * (rows_read + (m + 1) + m * (hb // 2) / hb)


# --------------------------------------------------------------------------
# CPU legs: the oracle port and the unmodified reference (test infrastructure;
# only these legs import oracle/ or baseline/_ref, never the product package)
# --------------------------------------------------------------------------
REF_TARGET = os.path.join(ROOT, "baseline", "_ref")


def _cpu_env():
    """lscpu model and the host's core count (state both)."""
    model = None
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cores": os.cpu_count(), "lscpu_model": model}


def _sweep_threaded(fn, nt, threads):
    """Run ``fn(lo, hi)`` over the reference's contiguous blocks
    (``parareal._block_bounds``, parareal.py:62-88) on a thread pool."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle.parareal import block_bounds as bb

    blocks = bb(nt, threads)
    if len(blocks) == 1:
        fn(*blocks[0])
        return
    with ThreadPoolExecutor(max_workers=len(blocks)) as pool:
        for f in [pool.submit(fn, lo, hi) for lo, hi in blocks]:
            f.result()


SETTINGS = {  # report the better of the two (threadpoolctl sets the BLAS pool)
    "threads=nproc, BLAS=1": lambda n: (n, 1),
    "threads=1, BLAS=nproc": lambda n: (1, n),
}


class CpuPort:
    """The oracle port (sine-Galerkin restatement of stepping.py:189-243 with
    dense numpy assembly + LAPACK solves) on a bounded sample of substeps of
    the bench workload, from the same inputs as the GPU arm: the coarse
    trajectory (oracle.run_coarse), i.e. the states of parareal's first sweep."""

    def __init__(self, cfg_id, P, slices=None, per_gpu=None):
        import oracle
        from oracle import problems as OP

        M, nt, m, alpha, T, tol = OP.CONFIG_GRIDS[cfg_id]
        self.cfg_id, self.M, self.m = cfg_id, M, m
        self.dims = 1 if cfg_id <= 3 else 2
        self.prob = OP.config(cfg_id)
        self.space = oracle.Sine1D(M) if self.dims == 1 else oracle.Sine2D(M, pcg_tol=1e-13)
        self.grids = oracle.TimeGrids(T, P, m)
        self.U = oracle.run_coarse(self.prob, self.space, self.grids)
        # 2-D oracle solves take seconds each: a sample of 8 slices
        self.slices = slices or (P if self.dims == 1 else min(P, 8))
        self.oracle = oracle
        self.sub = None

    def run(self, threads, blas, target_s):
        from threadpoolctl import threadpool_limits

        o = self.oracle

        def fn(lo, hi, sub):
            o.fine_sweep_intervals(self.U, lo, hi, self.space, self.grids, self.prob, substeps=sub)

        with threadpool_limits(limits=blas, user_api="blas"):
            if self.sub is None:  # size the sample once: ~target_s of CPU work
                t0 = time.perf_counter()
                _sweep_threaded(lambda lo, hi: fn(lo, hi, 1), self.slices, threads)
                per = time.perf_counter() - t0
                self.sub = max(1, min(self.m, int(target_s / max(per, 1e-9))))
            t0 = time.perf_counter()
            _sweep_threaded(lambda lo, hi: fn(lo, hi, self.sub), self.slices, threads)
            dt = time.perf_counter() - t0
        units = self.slices * self.sub
        return units * self.M ** self.dims / dt, dt

    def sample_text(self, setting):
        how = "dense numpy assembly + batched LU" if self.dims == 1 else "matrix-free numpy PCG, dense transforms"
        return (f"{self.slices} slices x the first {self.sub} of {self.m} substeps of config {self.cfg_id} "
                f"from the coarse trajectory (oracle sine-Galerkin port: {how}; {setting}); "
                f"extrapolated to the full sweep at the sampled rate")


class CpuReference:
    """The UNMODIFIED reference ``parafrac`` (baseline/_ref, pip-installed from
    /root/reference) on the Chebyshev form of a 1-D config (degree M+1: M
    interior unknowns, same P, alpha, T, D, f, u0 callbacks),
    through its own ``fine_sweep_intervals`` (stepping.py:189-243).  A bounded
    sample: the first ``sub`` substeps of every slice (grids with the config's
    dt and ``m = sub``), inputs the reference's own coarse trajectory."""

    def __init__(self, cfg_id, P):
        from oracle import problems as OP

        if not os.path.isdir(os.path.join(REF_TARGET, "parafrac")):
            raise RuntimeError("reference not installed under baseline/_ref")
        if REF_TARGET not in sys.path:
            sys.path.insert(0, REF_TARGET)
        import parafrac
        from parafrac import stepping

        M, nt, m, alpha, T, tol = OP.CONFIG_GRIDS[cfg_id]
        o = OP.config(cfg_id)
        self.pf, self.cfg_id, self.M, self.m, self.T, self.P = parafrac, cfg_id, M, m, T, P
        self.prob = parafrac.ProblemSpec(o.a, o.b, o.t_final, o.alpha, o.diffusion, o.source, o.initial,
                                         name=o.name)
        self.op = parafrac.build_operator(M + 1, 0.0, 1.0)
        self.U = stepping.run_coarse(self.prob, self.op, parafrac.TimeGrids(T, P, m))
        self.stepping = stepping
        self.sub = None

    def run(self, threads, blas, target_s):
        from threadpoolctl import threadpool_limits

        pf = self.pf

        def sweep(sub):
            g = pf.TimeGrids(self.T * sub / self.m, self.P, sub)  # the config's dt, first `sub` substeps

            def fn(lo, hi):
                self.stepping.fine_sweep_intervals(self.U, lo, hi, self.op, g, self.prob)

            _sweep_threaded(fn, self.P, threads)

        with threadpool_limits(limits=blas, user_api="blas"):
            if self.sub is None:
                t0 = time.perf_counter()
                sweep(1)
                per = time.perf_counter() - t0
                self.sub = max(1, min(self.m, int(target_s / max(per, 1e-9))))
            t0 = time.perf_counter()
            sweep(self.sub)
            dt = time.perf_counter() - t0
        return self.P * self.sub * self.M / dt, dt

    def sample_text(self, setting):
        return (f"{self.P} slices x the first {self.sub} of {self.m} substeps of config {self.cfg_id} in the "
                f"reference's Chebyshev form (degree {self.M + 1}), unmodified parafrac.fine_sweep_intervals "
                f"({setting}); extrapolated to the full sweep at the sampled rate")


def measure_cpu(leg, reps, target_s, warmup=1):
    """Both thread settings, min-of-reps after warm-up (harness.py:65-73):
    returns (best, per-setting results)."""
    n = os.cpu_count() or 1
    res = {}
    for name, mk in SETTINGS.items():
        threads, blas = mk(n)
        vals = []
        for i in range(warmup + reps):
            v, _ = leg.run(threads, blas, target_s)
            if i >= warmup:
                vals.append(v)
        res[name] = {"value": max(vals), "reps": len(vals), "sample": leg.sample_text(name)}
    best = max(res, key=lambda k: res[k]["value"])
    return best, res


def cpu_baseline_line(cfg_id, P, target_s, reps=3, with_reference=True):
    port = CpuPort(cfg_id, P)
    best, res = measure_cpu(port, reps, target_s)
    env = _cpu_env()
    out = {"value": res[best]["value"], "unit": "mode-steps/s", "cores": env["cores"], "kind": "port",
           "sample": res[best]["sample"], "setting": best, "settings": {k: v["value"] for k, v in res.items()},
           "lscpu_model": env["lscpu_model"], "extrapolated": True,
           "timing": f"max throughput over {reps} reps after 1 warm-up per setting (harness.py:65-73 min-time)"}
    if with_reference and cfg_id <= 3:
        try:
            ref = CpuReference(cfg_id, P)
            rbest, rres = measure_cpu(ref, reps, target_s)
            out["unmodified_reference"] = {"value": rres[rbest]["value"], "unit": "mode-steps/s",
                                           "setting": rbest, "sample": rres[rbest]["sample"],
                                           "settings": {k: v["value"] for k, v in rres.items()}}
        except Exception as exc:  # the installed reference is optional on the GPU arm
            out["unmodified_reference"] = {"unavailable": str(exc)}
    return out


def run_reference_arm(args, rank, world):
    """``--impl reference``: the reference's CPU path on the host cores (rank 0
    only; other ranks exit without work).  Each step is one bounded sample of
    the bench workload; warm-up and timed steps alternate the two thread
    settings; the line's value is the better setting's best step."""
    from oracle import problems as OP

    if rank != 0:
        return
    M, nt, m, alpha, T, tol = OP.CONFIG_GRIDS[args.config]
    dims = 1 if args.config <= 3 else 2
    P_rank = 64 if args.config == 5 else nt
    port = CpuPort(args.config, P_rank * world)
    n = os.cpu_count() or 1
    names = list(SETTINGS)
    per = {k: [] for k in names}
    for i in range(args.warmup + args.steps):
        name = names[i % 2]
        threads, blas = SETTINGS[name](n)
        v, _ = port.run(threads, blas, args.ref_seconds)
        if i >= args.warmup:
            per[name].append(v)
    best = max((k for k in names if per[k]), key=lambda k: max(per[k]))
    v = max(per[best])
    units = P_rank * m * M ** dims
    env = _cpu_env()
    cpu = {"value": v, "unit": "mode-steps/s", "cores": env["cores"], "kind": "port",
           "sample": port.sample_text(best), "setting": best,
           "settings": {k: (max(x) if x else None) for k, x in per.items()}, "lscpu_model": env["lscpu_model"],
           "extrapolated": True}
    if dims == 1:
        try:
            ref = CpuReference(args.config, P_rank * world)
            rbest, rres = measure_cpu(ref, 2, args.ref_seconds)
            cpu["unmodified_reference"] = {"value": rres[rbest]["value"], "unit": "mode-steps/s",
                                           "setting": rbest, "sample": rres[rbest]["sample"],
                                           "settings": {k: x["value"] for k, x in rres.items()}}
        except Exception as exc:
            cpu["unmodified_reference"] = {"unavailable": str(exc)}
    line = {
        "impl": "reference", "metric": "fine mode-steps/s", "value": v, "unit": "mode-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * units / v,
        "ms_per_step_note": "extrapolated: one full sweep at the best sampled rate (each step times a "
                            "bounded sample of substeps, see cpu_baseline.sample)",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config RNG convention, SURVEY.md §8d)",
        "config": _config_dict(args.config, world, P_rank),
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "mode-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(cfg_id, world, per_gpu):
    from oracle import problems as OP

    M, nt, m, alpha, T, tol = OP.CONFIG_GRIDS[cfg_id]
    dims = 1 if cfg_id <= 3 else 2
    return {"workload": f"config{cfg_id}: {dims}-D sine Galerkin fine sweep", "modes": M,
            "slices_per_gpu": per_gpu, "slices_total": per_gpu * world, "fine_steps_per_slice": m,
            "alpha": alpha, "t_final": T, "parallelism": f"slices sharded over {world} GPU(s)",
            "l2": "inputs larger than L2 (history paths > 126 MB)" if cfg_id >= 3 else "inputs fit in L2",
            "inputs": "coarse trajectory (run_coarse): the states of parareal's first fine sweep"}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def _parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parareal", action="store_true")
    ap.add_argument("--slices", type=int, default=None,
                    help="slices per GPU (default: the config's P; config 5: 512 at one GPU, 64 per GPU above)")
    ap.add_argument("--tiled-u0", action="store_true",
                    help="sweep inputs: the initial state in every slice instead of the coarse trajectory")
    ap.add_argument("--dist", action="store_true",
                    help="use the torch.distributed (NCCL) driver even at one rank (exercises the multi-GPU path)")
    return ap.parse_args()


def _slices_per_gpu(args, world):
    from oracle import problems as OP

    if args.slices:
        return args.slices
    P = OP.CONFIG_GRIDS[args.config][1]
    if args.config == 5:
        # BASELINE config 5: P = 512 slices, 64 per GPU at 8 GPUs; one GPU runs the whole problem
        return 512 if world == 1 else 64
    return P


def _gpu_arm(args, rank, world, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1 or args.dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2510_11023_b200 as pfb
    from paper_2510_11023_b200 import _lib
    from paper_2510_11023_b200.parallel import block_bounds
    from paper_2510_11023_b200.problems import CONFIGS

    cfg = CONFIGS[args.config]
    M, m = cfg["modes"], cfg["m"]
    dims = cfg["dims"]
    P_rank = _slices_per_gpu(args, world)
    P = P_rank * world
    prob = pfb.config_problem(args.config)
    op = pfb.build_sine_operator(M, dims=dims)
    grids = pfb.TimeGrids(cfg["t_final"], P, m)
    lo, hi = block_bounds(P, world)[rank]
    # a context of its own (not the public API's cache): its stream binding stays here
    ctx = _lib.Context(prob, op, grids, device=local)
    stream = torch.cuda.Stream(device=local)
    _lib.lib.pf_set_stream(ctx.handle, _lib.C.c_void_p(stream.cuda_stream))

    # untimed inputs of the sweep: the coarse trajectory, i.e. the states of
    # parareal's first fine sweep (--tiled-u0: every slice from the initial state)
    traj = (np.tile(pfb.initial_state(prob, op), (P + 1, 1)) if args.tiled_u0
            else pfb.run_coarse(prob, op, grids))
    with torch.cuda.stream(stream):
        U = torch.from_numpy(traj).to(f"cuda:{local}")
        out = torch.empty((hi - lo, M ** dims), dtype=torch.float64, device=f"cuda:{local}")
    stream.synchronize()

    def step():
        ctx.check(_lib.lib.pf_dev_fine_sweep_async(ctx.handle, _lib.C.c_void_p(U.data_ptr()), lo, hi,
                                                   _lib.C.c_void_p(out.data_ptr())))

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.check(_lib.lib.pf_dev_check(ctx.handle))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.stats()["kernel_launches"]
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ctx.check(_lib.lib.pf_dev_check(ctx.handle))
    launches = ctx.stats()["kernel_launches"] - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    units_total = P * m
    value = units_total * M ** dims / (ms / 1e3)

    # per-launch work counters: one more (untimed) launch decoded on its own
    _lib.lib.pf_reset_stats(ctx.handle)
    step()
    ctx.check(_lib.lib.pf_dev_check(ctx.handle))
    st = ctx.stats()
    flops = (sweep_flops(M, m, hi - lo, lo, st["pcg_iterations"], st["solves"]) if dims == 1
             else sweep_flops_2d(M, m, hi - lo, lo, st["pcg_iterations"]))
    achieved_tf = flops / (ms / 1e3) / 1e12
    # far-history engine of this size: the grouped TMA-fed DMMA helper at M = 512 (1-D), unless overridden
    hist_group = 4 if (dims == 1 and M == 512 and os.environ.get("PF_FAR_TC", "2") == "2") else 1
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6547.5)
    roof = {"bound": "fp64", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": None,
            "bound_note": "FP64 pipe (DFMA in the slice CTAs, DMMA.8x8x4 in the helper CTAs; both measured at the "
                          "same rate on this pool): FP64 has no tcgen05 kind, so the binding compute roof is the "
                          "FP64 peak, not the bf16 tensor figure",
            "peak_source": "measured FP64 DMMA/DFMA peak (profiles/fp64_peaks_r01.txt); "
                           "MEASURED_PEAKS.json has HBM and bf16 only",
            "flops_per_launch": flops, "pcg_iterations_per_launch": st["pcg_iterations"],
            "solves_per_launch": st["solves"],
            "pcg_iterations_per_solve": st["pcg_iterations"] / max(st["solves"], 1),
            "hbm_bytes_per_launch_model": history_bytes(M ** dims, m, hi - lo, group=hist_group),
            "hbm_peak_gbs": hbm_peak,
            "hbm_frac_model": history_bytes(M ** dims, m, hi - lo, group=hist_group) / (ms / 1e3) / 1e9 / hbm_peak}
    try:
        with open(os.path.join(ROOT, "profiles", f"dram_config{args.config}.json")) as f:
            dram = json.load(f)
        roof["traffic"] = dram.get("dram_bytes_per_step")
        roof["traffic_source"] = dram.get("source")
        if roof["traffic"]:
            roof["hbm_frac_measured_traffic"] = roof["traffic"] / (ms / 1e3) / 1e9 / hbm_peak
    except OSError:
        pass

    # e2e through the public API with pinned host buffers (H2D + kernel + D2H each step)
    host_U = torch.empty(traj.shape, dtype=torch.float64, pin_memory=True).numpy()
    host_U[:] = traj
    pfb.fine_sweep_intervals(host_U, lo, hi, op, grids, prob)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pfb.fine_sweep_intervals(host_U, lo, hi, op, grids, prob)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": units_total * M ** dims / e2e_s, "unit": "mode-steps/s",
           "h2d_bytes_per_step": int(hi * M ** dims * 8), "d2h_bytes_per_step": int((hi - lo) * M ** dims * 8),
           "api": "paper_2510_11023_b200.fine_sweep_intervals (ctypes -> pf_fine_sweep)"}

    parareal = None
    if not args.no_parareal and not dist.is_initialized():
        # one untimed solve (the driver's buffers and streams are allocated on first use), then
        # the minimum of three timed solves (the reference harness's convention, harness.py:65-73);
        # the 2-D configs run for seconds: one timed solve
        reps = 3 if dims == 1 else 1
        times = []
        for rep_i in range(reps + (1 if dims == 1 else 0)):
            t0 = time.perf_counter()
            it, rep = pfb.parareal_solve(prob, op, grids, tol=cfg["tol"], k_max=P + 1)
            times.append(time.perf_counter() - t0)
        timed = times[1:] if dims == 1 else times
        parareal = {"time_to_tol_s": min(timed), "iterations": rep.iterations,
                    "stop_reason": rep.stop_reason, "final_diff": rep.diffs[-1], "slices": P,
                    "first_call_s": times[0], "timed_solves_s": timed,
                    "note": "public API parareal_solve, initial coarse sweep + all iterations; "
                            + ("min of 3 after one untimed solve" if dims == 1 else "one solve")}
    elif not args.no_parareal:
        # multi-GPU time-to-tol: slices sharded over the ranks, one NCCL all-gather
        # of the fine endpoints per iteration, replicated correction (parallel.py)
        from paper_2510_11023_b200.parallel import DeviceOps, DistributedParareal
        dp = DistributedParareal(DeviceOps(prob, op, grids, local), P)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = dp.solve(tol=cfg["tol"], k_max=P + 1)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        parareal = {"time_to_tol_s": float(t.item()), "iterations": res["k"], "stop_reason": res["stop_reason"],
                    "final_diff": res["diffs"][-1], "slices": P,
                    "note": f"parallel.DistributedParareal over {world} ranks (NCCL all-gather of F_old per "
                            "iteration), initial coarse sweep + all iterations, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.config, P, target_s=args.ref_seconds, reps=2)

    if rank == 0:
        line = {
            "metric": "fine mode-steps/s", "value": value, "unit": "mode-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config RNG convention, SURVEY.md §8d)",
            "config": dict(_config_dict(args.config, world, P_rank),
                           **({"inputs": "initial state in every slice (--tiled-u0)"} if args.tiled_u0 else {})),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "parareal": parareal,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def _spawned(local, args, world, port):
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    _gpu_arm(args, local, world, local)


def main():
    args = _parse()
    if "WORLD_SIZE" in os.environ:  # under torchrun: one process per GPU already
        world = int(os.environ["WORLD_SIZE"])
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
    else:
        world, rank, local = max(1, args.gpus), 0, 0
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without torchrun: spawn one process per GPU (NCCL, 127.0.0.1)
        import socket

        import torch.multiprocessing as mp

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        mp.spawn(_spawned, args=(args, world, port), nprocs=world, join=True)
        return
    _gpu_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
