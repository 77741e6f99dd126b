"""Multi-rank parareal driver (paper_2510_11023_b200.parallel) under gloo on CPU.

The GPU ranks run the sm_100a sweep; here each rank runs the oracle sweep on
CPU tensors behind the same ops interface, so the sharding
(parareal._block_bounds, parareal.py:62-72), the padded all-gather with
uneven blocks, the G_old reuse, the frozen-prefix skip of unchanged slices
and the replicated correction sweep are
checked for world_size 2 and 3 against the single-process oracle —
iterates must agree bitwise (the rank-count analogue of the reference's
thread-count invariance, test_parareal.py:128-138).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import problems as P
from paper_2510_11023_b200.parallel import DistributedParareal, block_bounds


class OracleOps:
    """CPU stand-in for DeviceOps: same state machine, oracle arithmetic."""

    torch = torch

    def __init__(self, problem, space, grids, block_lo=0):
        self.problem, self.space, self.grids = problem, space, grids
        self.size = space.size
        # the oracle's batched numpy sweep is not bitwise batch-composition
        # invariant (the device kernel is: one CTA per slice), so a partial
        # sweep [lo, hi) recomputes the rank's whole block and keeps the tail
        self.block_lo = block_lo

    def empty(self, rows):
        return torch.empty((rows, self.size), dtype=torch.float64)

    def init(self):
        self.U = oracle.run_coarse(self.problem, self.space, self.grids)
        self.gold = self.U[1:].copy()
        self.gnew = np.empty_like(self.gold)
        self.k = -1

    def fine(self, lo, hi, out):
        self.swept = getattr(self, "swept", 0) + (hi - lo)
        full = oracle.fine_sweep_intervals(self.U, self.block_lo, hi, self.space, self.grids, self.problem)
        out[: hi - lo] = torch.from_numpy(full[lo - self.block_lo:])

    def correct(self, fold_all, k):
        if k > 0:
            self.gold, self.gnew = self.gnew, self.gold
        fold = fold_all.numpy()
        nxt = np.empty_like(self.U)
        nxt[0] = self.U[0]
        for n in range(self.grids.nt):
            self.gnew[n] = oracle.coarse_step(nxt[: n + 1], self.space, self.grids, self.problem, step_index=n)
            nxt[n + 1] = fold[n] + (self.gnew[n] - self.gold[n])
        diff = max(self.space.norm(nxt[n] - self.U[n]) for n in range(self.grids.nt + 1))
        same = [np.array_equal(nxt[n].view(np.int64), self.U[n].view(np.int64)) for n in range(self.grids.nt + 1)]
        self.first_changed = same.index(False) if False in same else self.grids.nt
        self.U = nxt
        return diff

    def frozen(self):
        return self.first_changed

    def read(self):
        return self.U, self.gnew, self.gold


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nt, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = P.config(1, modes=8)
        ops = OracleOps(prob, oracle.Sine1D(8), oracle.TimeGrids(1.0, nt, 4), block_bounds(nt, world)[rank][0])
        res = DistributedParareal(ops, nt).solve(tol=1e-12, k_max=nt + 1)
        out_q.put((rank, res["states"], res["diffs"], res["k"], res["coarse_old"], res["fine_endpoints"],
                   getattr(ops, "swept", 0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nt", [(2, 5), (3, 7)])
def test_distributed_matches_single_process(world, nt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nt, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = P.config(1, modes=8)
    sp = oracle.Sine1D(8)
    it, rep = oracle.solve(prob, sp, oracle.TimeGrids(1.0, nt, 4), tol=1e-12, k_max=nt + 1)
    swept = 0
    for rank, states, diffs, k, g_old, f_old, sw in results:
        swept += sw
        assert k == rep.iterations
        np.testing.assert_array_equal(states, it.states)
        np.testing.assert_array_equal(g_old, it.coarse_old)
        np.testing.assert_array_equal(f_old, it.fine_endpoints)
        assert diffs == rep.diffs
    # iteration k re-sweeps only slices k..nt-1 (the frozen prefix is skipped)
    assert swept == sum(nt - k for k in range(rep.iterations)), (swept, rep.iterations)


def test_uneven_bounds_cover_all_ranks():
    b = block_bounds(5, 3)
    assert b == [(0, 2), (2, 4), (4, 5)]
