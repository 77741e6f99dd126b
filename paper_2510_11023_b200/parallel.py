"""Multi-GPU parareal: one process per GPU, slices sharded across ranks.

The reference's only parallelism is a thread pool over contiguous slice
blocks (``parareal.py:62-88``).  Here the same contiguous rule
(``block_bounds`` == ``_block_bounds``) assigns slices to ranks; per
iteration every rank

1. runs the fine sweep of its block on its GPU (one kernel launch),
2. all-gathers the fine endpoints F_old over NCCL (the only exchange: no
   fine history ever crosses slices),
3. runs the identical, deterministic sequential correction sweep
   (``parareal.py:114-128``) on its own GPU, so every rank holds the same
   iterate without a broadcast.

Results are bitwise independent of the rank count because each slice's sweep
is the same kernel arithmetic whatever block it is launched in, and the
correction runs on the full gathered F_old.  ``DeviceOps`` drives the C-ABI;
tests substitute CPU ops to check the sharding and exchange logic under
``gloo``.
"""

from __future__ import annotations

import contextlib
import time

import numpy as np

__all__ = ["DeviceOps", "DistributedParareal", "block_bounds"]


def block_bounds(count, parts):
    """Contiguous, near-even split of ``range(count)`` (``parareal.py:62-72``)."""
    blocks = min(parts, count)
    base, extra = divmod(count, blocks)
    bounds, lo = [], 0
    for i in range(blocks):
        hi = lo + base + (1 if i < extra else 0)
        bounds.append((lo, hi))
        lo = hi
    return bounds


class DeviceOps:
    """Per-rank device state machine over ``pf_dev_parareal_*`` (C-ABI).

    Owns its context (not the process-wide cache: the state machine's buffers
    and stream binding must not leak into other callers) and a stream; the
    driver runs inside ``scope()``, which makes that stream torch's current
    stream only for the duration of the solve, so kernels, NCCL and copies
    stay ordered without changing the caller's stream afterwards.
    """

    def __init__(self, problem, op, grids, device):
        import torch

        from . import _lib
        from .spaces import initial_state

        self.torch = torch
        self._lib = _lib
        self.device = torch.device("cuda", device)
        self.ctx = _lib.Context(problem, op, grids, device=device)
        self.size = op.interior_size
        self.nt = grids.nt
        self.u0 = _lib.f64(initial_state(problem, op))
        self.stream = torch.cuda.Stream(device=self.device)
        _lib.lib.pf_set_stream(self.ctx.handle, _lib.C.c_void_p(self.stream.cuda_stream))

    def scope(self):
        return self.torch.cuda.stream(self.stream)

    def empty(self, rows):
        return self.torch.empty((rows, self.size), dtype=self.torch.float64, device=self.device)

    def init(self):
        L = self._lib
        self.ctx.check(L.lib.pf_dev_parareal_init(self.ctx.handle, L.ptr(self.u0)))

    def fine(self, lo, hi, out):
        L = self._lib
        states = L.lib.pf_dev_parareal_states(self.ctx.handle)
        self.ctx.check(L.lib.pf_dev_fine_sweep(self.ctx.handle, L.C.c_void_p(states), lo, hi,
                                               L.C.c_void_p(out.data_ptr())))

    def frozen(self):
        """Leading nodes the last correction left bitwise unchanged."""
        return int(self._lib.lib.pf_dev_parareal_frozen(self.ctx.handle))

    def correct(self, fold_all, k):
        L = self._lib
        diff = L.C.c_double(0.0)
        self.ctx.check(L.lib.pf_dev_parareal_correct(self.ctx.handle, L.C.c_void_p(fold_all.data_ptr()), int(k),
                                                     L.C.byref(diff)))
        return float(diff.value)

    def read(self):
        L = self._lib
        states = np.empty((self.nt + 1, self.size))
        g_new = np.empty((self.nt, self.size))
        g_old = np.empty((self.nt, self.size))
        self.ctx.check(L.lib.pf_dev_parareal_read(self.ctx.handle, L.ptr(states), L.ptr(g_new), L.ptr(g_old)))
        return states, g_new, g_old


class DistributedParareal:
    """Parareal over ``world`` ranks of an initialised ``torch.distributed`` group."""

    def __init__(self, ops, nt, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.ops = ops
        self.nt = nt
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.bounds = block_bounds(nt, self.world)
        # ranks beyond the slice count own nothing but still take part in the gather
        while len(self.bounds) < self.world:
            self.bounds.append((nt, nt))
        self.chunk = max(hi - lo for lo, hi in self.bounds)

    def gather(self, local):
        """All-gather uneven blocks: pad to the largest block, gather, compact."""
        torch = self.ops.torch
        lo, hi = self.bounds[self.rank]
        send = self.ops.empty(self.chunk)
        if hi > lo:
            send[: hi - lo].copy_(local[: hi - lo])
        if not self.dist.is_initialized():
            return send[: hi - lo]
        recv = self.ops.empty(self.chunk * self.world)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)
        parts = [recv[r * self.chunk: r * self.chunk + (b - a)] for r, (a, b) in enumerate(self.bounds)]
        return torch.cat(parts, dim=0).contiguous()

    def solve(self, tol=1e-10, k_max=20):
        """``parareal.py:91-155`` across ranks; returns the reference's result fields."""
        scope = getattr(self.ops, "scope", None)
        with (scope() if scope is not None else contextlib.nullcontext()):
            return self._solve(tol, k_max)

    def _solve(self, tol, k_max):
        t0 = time.perf_counter()
        self.ops.init()
        lo, hi = self.bounds[self.rank]
        local = self.ops.empty(max(hi - lo, 1))
        diffs, times, fold = [], [], None
        stop_reason, iterations = "k_max", 0
        for k in range(k_max):
            # slices below the frozen prefix keep their F_old rows (their inputs
            # are bitwise those of their last sweep): finite termination made exact
            start = lo if k == 0 else max(lo, min(hi, self.ops.frozen()))
            if hi > start:
                self.ops.fine(start, hi, local[start - lo:])
            fold = self.gather(local)
            diff = self.ops.correct(fold, k)
            diffs.append(diff)
            times.append(time.perf_counter() - t0)
            iterations = k + 1
            if tol is not None and diff < tol:
                stop_reason = "tol"
                break
        states, g_new, g_old = self.ops.read()
        f_old = fold.cpu().numpy() if fold is not None else None
        return {"k": iterations, "states": states, "coarse_new": g_new, "coarse_old": g_old,
                "fine_endpoints": f_old, "diffs": diffs, "iteration_times": times,
                "stop_reason": stop_reason, "wall_time": time.perf_counter() - t0,
                "world": self.world}
