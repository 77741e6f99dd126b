#!/usr/bin/env python
"""Benchmark of the parareal fine-propagator sweep (BASELINE.json metric).

One *step* is one fine sweep (``fine_sweep_intervals``, stepping.py:189-243)
over every slice a GPU owns, with the coarse states already resident in HBM.
Default workload: BASELINE config 3 (1-D sine Galerkin, M=512, P=64 slices,
m=1024 fine steps per slice, alpha=0.3, T=2) — the largest 1-D config and the
first on which a roofline binds; config 2 (``configs[1]``) is
latency-bound with 16 slices and is a parity case.  ``--config`` selects 1-3.

    python bench.py [--gpus N --steps K --warmup W --config 3]
    python bench.py --impl reference ...      # CPU arm: the oracle port on the host cores

Under torchrun (N > 1) each rank sweeps its contiguous block of a global
problem with P*N slices (parareal._block_bounds, parareal.py:62-72): weak
scaling, no collective inside the sweep.  Timing: CUDA events on the launch
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


def history_bytes(M, m, slices, hb=8):
    """HBM bytes of the blocked history: each path row read once per block + written once."""
    rows_read = sum(((r0 + 1)) for r0 in range(0, m, hb))
    return slices * 8.0 * M * (rows_read + (m + 1) + m * (hb // 2) / hb)


# --------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy sine-Galerkin restatement of stepping.py)
# --------------------------------------------------------------------------
def cpu_sample(cfg_id, nt, target_s=15.0, lo=0, hi=None):
    import oracle
    from paper_2510_11023_b200.problems import CONFIGS, config_problem

    cfg = CONFIGS[cfg_id]
    M, m = cfg["modes"], cfg["m"]
    hi = nt if hi is None else hi
    prob = config_problem(cfg_id)
    dims = cfg["dims"]
    space = oracle.Sine1D(M) if dims == 1 else oracle.Sine2D(M, pcg_tol=cfg.get("pcg_tol", 1e-13))
    grids = oracle.TimeGrids(cfg["t_final"], nt, m)
    # the sample's timing does not depend on the coarse states: every slice
    # starts from the initial state (no coarse sweep on the CPU)
    u0 = space.initial_state(prob)
    U = np.tile(u0, (nt + 1, 1))
    if dims == 2:
        hi = min(hi, lo + 4)  # 2-D oracle solves cost seconds each: sample 4 slices
    t0 = time.perf_counter()
    oracle.fine_sweep_intervals(U, lo, hi, space, grids, prob, substeps=1)
    per = time.perf_counter() - t0
    sub = max(1, min(m, int(target_s / max(per, 1e-9))))
    t0 = time.perf_counter()
    oracle.fine_sweep_intervals(U, lo, hi, space, grids, prob, substeps=sub)
    dt = time.perf_counter() - t0
    units = (hi - lo) * sub
    how = ("dense numpy assembly + batched LU" if dims == 1 else "matrix-free numpy PCG, dense transforms")
    return {"value": units * M ** dims / dt, "unit": "mode-steps/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{hi - lo} slices x {sub} of {m} substeps of config {cfg_id} "
                      f"(oracle sine-Galerkin port: {how}, OpenBLAS threads)",
            "seconds": dt}


def run_reference_arm(args, rank, world):
    from paper_2510_11023_b200.problems import CONFIGS

    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    P = cfg["nt"] * world
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_sample(args.config, P, target_s=args.ref_seconds,
                               lo=0, hi=cfg["nt"]))
    vals = vals[args.warmup:]
    v = statistics.median(x["value"] for x in vals)
    ms = 1e3 * cfg["nt"] * cfg["m"] * cfg["modes"] ** cfg["dims"] / v
    line = {
        "impl": "reference", "metric": "fine mode-steps/s", "value": v, "unit": "mode-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config RNG convention, SURVEY.md §8d)",
        "config": _config_dict(args.config, world),
        "cpu_baseline": {k: vals[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
        "e2e": {"value": v, "unit": "mode-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(cfg_id, world, per_gpu=None):
    from paper_2510_11023_b200.problems import CONFIGS

    cfg = dict(CONFIGS[cfg_id])
    if per_gpu is not None:
        cfg["nt"] = per_gpu
    return {"workload": f"config{cfg_id}: {cfg['dims']}-D sine Galerkin fine sweep", "modes": cfg["modes"],
            "slices_per_gpu": cfg["nt"], "slices_total": cfg["nt"] * world, "fine_steps_per_slice": cfg["m"],
            "alpha": cfg["alpha"], "t_final": cfg["t_final"], "parallelism": f"slices sharded over {world} GPU(s)",
            "l2": "inputs larger than L2 (history paths > 126 MB)" if cfg_id >= 3 else "inputs fit in L2",
            "inputs": "coarse trajectory (run_coarse): the states of parareal's first fine sweep"}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parareal", action="store_true")
    ap.add_argument("--tiled-u0", action="store_true",
                    help="sweep inputs: the initial state in every slice instead of the coarse trajectory")
    ap.add_argument("--dist", action="store_true",
                    help="use the torch.distributed (NCCL) driver even at one rank (exercises the multi-GPU path)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

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
    M, m, P_rank = cfg["modes"], cfg["m"], cfg["nt"]
    dims = cfg["dims"]
    if args.config == 5 and world == 1:
        P_rank = 64  # config 5 is the scaling run: 64 slices per GPU (BASELINE.json)
    P = P_rank * world
    prob = pfb.config_problem(args.config)
    op = pfb.build_sine_operator(M, dims=dims)
    grids = pfb.TimeGrids(cfg["t_final"], P, m)
    lo, hi = block_bounds(P, world)[rank]
    ctx = _lib.context_for(prob, op, grids, device=local)
    # one dedicated stream: the kernels and the timing events share it
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    _lib.lib.pf_set_stream(ctx.handle, _lib.C.c_void_p(stream.cuda_stream))

    # untimed inputs of the sweep: the coarse trajectory, i.e. the states of
    # parareal's first fine sweep (--tiled-u0: every slice from the initial state)
    traj = (np.tile(pfb.initial_state(prob, op), (P + 1, 1)) if args.tiled_u0
            else pfb.run_coarse(prob, op, grids))
    U = torch.from_numpy(traj).to(f"cuda:{local}")
    out = torch.empty((hi - lo, M ** dims), dtype=torch.float64, device=f"cuda:{local}")

    def step():
        ctx.check(_lib.lib.pf_dev_fine_sweep_async(ctx.handle, _lib.C.c_void_p(U.data_ptr()), lo, hi,
                                                   _lib.C.c_void_p(out.data_ptr())))

    for _ in range(max(args.warmup, 1)):
        step()
    ctx.check(_lib.lib.pf_dev_check(ctx.handle))
    _lib.lib.pf_reset_stats(ctx.handle)
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
    ctx.check(_lib.lib.pf_dev_check(ctx.handle))  # decodes the last launch's status (+ its counters)
    st = ctx.stats()
    launches = st["kernel_launches"] - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    units_total = P * m
    value = units_total * M ** dims / (ms / 1e3)

    # roofline of the dominant (only) kernel in the step
    flops = (sweep_flops(M, m, hi - lo, lo, st["pcg_iterations"], st["solves"]) if dims == 1
             else sweep_flops_2d(M, m, hi - lo, lo, st["pcg_iterations"]))
    achieved_tf = flops / (ms / 1e3) / 1e12
    peaks = _peaks()
    roof = {"bound": "tensor", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": None,
            "peak_source": "measured FP64 DMMA/DFMA peak (profiles/fp64_peaks_r01.txt); "
                           "MEASURED_PEAKS.json has HBM and bf16 only",
            "flops_per_launch": flops, "pcg_iterations_per_launch": st["pcg_iterations"],
            "pcg_iterations_per_solve": st["pcg_iterations"] / max(st["solves"], 1),
            "hbm_bytes_per_launch": history_bytes(M ** dims, m, hi - lo),
            "hbm_frac": history_bytes(M ** dims, m, hi - lo) / (ms / 1e3) / 1e9 / peaks.get("hbm_gbs", 6537.0)}
    try:
        with open(os.path.join(ROOT, "profiles", f"dram_config{args.config}.json")) as f:
            dram = json.load(f)
        roof["traffic"] = dram.get("dram_bytes_per_launch")
        if dram.get("dominant_kernel"):
            roof["dominant_kernel"] = dram["dominant_kernel"]
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
        res = pfb.fine_sweep_intervals(host_U, lo, hi, op, grids, prob)
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
        t0 = time.perf_counter()
        it, rep = pfb.parareal_solve(prob, op, grids, tol=cfg["tol"], k_max=P + 1)
        parareal = {"time_to_tol_s": time.perf_counter() - t0, "iterations": rep.iterations,
                    "stop_reason": rep.stop_reason, "final_diff": rep.diffs[-1],
                    "note": "public API parareal_solve, initial coarse sweep + all iterations"}
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
                    "final_diff": res["diffs"][-1],
                    "note": f"parallel.DistributedParareal over {world} ranks (NCCL all-gather of F_old per "
                            "iteration), initial coarse sweep + all iterations, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.config, P, target_s=15.0)
        cpu.pop("seconds", None)

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


if __name__ == "__main__":
    main()
