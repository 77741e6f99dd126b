"""The multi-rank driver on real devices: ``DistributedParareal`` over
``DeviceOps`` with NCCL, one process per GPU (``parareal.py:62-88`` sharded
over ranks).  Needs >= 2 GPUs (the driver's multi-GPU node); on a single-GPU
box it is skipped — the same sharding, padded all-gather, frozen-prefix skip
and replicated correction are covered on CPU by tests/test_distributed.py
(gloo, world sizes 2 and 3)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_2510_11023_b200 as pfb
        from paper_2510_11023_b200.parallel import DeviceOps, DistributedParareal

        modes, nt, m, dims = cfg
        prob = pfb.config_problem(3 if dims == 1 else 4, modes=modes)
        op = pfb.build_sine_operator(modes, dims=dims)
        g = pfb.TimeGrids(2.0 if dims == 1 else 1.0, nt, m)
        res = DistributedParareal(DeviceOps(prob, op, g, rank), nt).solve(tol=1e-12, k_max=nt + 1)
        q.put((rank, res["k"], res["states"], res["fine_endpoints"], res["diffs"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [(64, 12, 32, 1), (16, 6, 8, 2)])
def test_nccl_ranks_match_single_gpu(cfg):
    import torch
    import torch.multiprocessing as mp

    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs (multi-rank NCCL); CPU coverage: tests/test_distributed.py")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import paper_2510_11023_b200 as pfb

    modes, nt, m, dims = cfg
    prob = pfb.config_problem(3 if dims == 1 else 4, modes=modes)
    op = pfb.build_sine_operator(modes, dims=dims)
    g = pfb.TimeGrids(2.0 if dims == 1 else 1.0, nt, m)
    it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=nt + 1)
    for rank, k, states, f_old, diffs in results:
        assert k == rep.iterations
        # GPU-count invariance (the device analogue of test_parareal.py:128-138):
        # per-slice kernel arithmetic does not depend on the block a slice is swept in
        np.testing.assert_array_equal(states, it.states)
        np.testing.assert_array_equal(f_old, it.fine_endpoints)
        assert diffs == rep.diffs


@pytest.mark.parametrize("cfg,world", [((64, 12, 32, 1), 2), ((64, 12, 32, 1), 3), ((16, 6, 8, 2), 2)])
def test_rank_state_machines_on_one_gpu(cfg, world):
    """The per-rank device path of the multi-GPU driver on one B200: `world`
    DeviceOps contexts (one per rank), each sweeping its parareal._block_bounds
    block (pf_dev_fine_sweep with n_lo > 0, the per-rank frozen prefix, the 2-D
    warm starts indexed by global slice), exchanged through the host instead of
    NCCL and run one after the other (no rank waits on another inside a
    kernel).  Every rank must hold bitwise the single-process iterate."""
    import torch

    import paper_2510_11023_b200 as pfb
    from paper_2510_11023_b200.parallel import DeviceOps, block_bounds

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a B200")
    modes, nt, m, dims = cfg
    prob = pfb.config_problem(3 if dims == 1 else 4, modes=modes)
    op = pfb.build_sine_operator(modes, dims=dims)
    g = pfb.TimeGrids(2.0 if dims == 1 else 1.0, nt, m)
    it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=nt + 1)
    bounds = block_bounds(nt, world)
    ranks = [DeviceOps(prob, op, g, 0) for _ in range(world)]
    for ops in ranks:
        with ops.scope():
            ops.init()
    locals_ = [ops.empty(max(hi - lo, 1)) for ops, (lo, hi) in zip(ranks, bounds)]
    diffs = []
    for k in range(nt + 1):
        for ops, (lo, hi), loc in zip(ranks, bounds, locals_):
            with ops.scope():
                start = lo if k == 0 else max(lo, min(hi, ops.frozen()))
                if hi > start:
                    ops.fine(start, hi, loc[start - lo:])
                ops.stream.synchronize()
        fold = torch.cat([loc[: hi - lo] for loc, (lo, hi) in zip(locals_, bounds)], dim=0).contiguous()
        ds = []
        for ops in ranks:
            with ops.scope():
                ds.append(ops.correct(fold.to(ops.device), k))
        assert all(d == ds[0] for d in ds)  # the replicated correction agrees bitwise
        diffs.append(ds[0])
        if ds[0] < 1e-12:
            break
    assert len(diffs) == rep.iterations and diffs == rep.diffs
    for ops in ranks:
        with ops.scope():
            states, g_new, g_old = ops.read()
        np.testing.assert_array_equal(states, it.states)
        np.testing.assert_array_equal(g_new, it.coarse_new)
    np.testing.assert_array_equal(fold.cpu().numpy(), it.fine_endpoints)
