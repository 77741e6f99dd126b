"""Full-mode 2-D oracle runs (configs 4-5) for the device parity tests — TEST
INFRASTRUCTURE ONLY (CPU, long).

    python tests/golden/make_oracle_2d.py 4              # config 4 at full size, run to tol (~1 h on 8 cores)
    python tests/golden/make_oracle_2d.py 5 --nt 16      # config 5, 256^2 modes, P = 16 slices (reduced P)

The oracle is ``oracle.parareal`` (the restatement of ``parareal.py:91-155`` /
``stepping.py:124-243`` with ``oracle.Sine2D``, PCG tol 1e-13, guess = the
previous state).  The only change here is *where* the fine sweeps run: the
reference's own ``_parallel_stage`` (``parareal.py:75-88``) splits the slices
into contiguous blocks and runs them on a thread pool; this script runs the
same blocks in worker processes (OpenBLAS single-threaded).  The reference
asserts block-split invariance bitwise (``test_stepping.py:166-175``), and
``oracle.block_bounds`` is its rule, so the iterate is the serial one.

Fixture (``tests/golden/oracle_cfg<i>_2d[_nt<P>].npz``), sized for git:
  nodes            node indices stored in full (every ``stride``-th, default P/8, and the last)
  states, fine     the final iterate and F_old at those nodes
  states_k2        the iterate after iteration 2 at those nodes
  proj             every node of the final iterate projected on 8 seeded
                   Gaussian vectors (catches a mismatch at any node)
  norms            Euclidean norm of every node of the final iterate
  diffs, iterations, stop, pcg_mean
"""

import argparse
import os
import sys
import time
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from oracle import problems as P  # noqa: E402
from oracle import stepping as S  # noqa: E402
from oracle.parareal import DIVERGENCE_FACTOR, block_bounds  # noqa: E402

_W = {}


def _init(i, M, nt, m, T):
    _W["prob"] = P.config(i)
    _W["space"] = oracle.Sine2D(M, pcg_tol=1e-13)
    _W["grids"] = oracle.TimeGrids(T, nt, m)


def _block(args):
    U, lo, hi = args
    sp, gr, pb = _W["space"], _W["grids"], _W["prob"]
    sp.pcg_iterations.clear()
    f = S.fine_sweep_intervals(U, lo, hi, sp, gr, pb)
    g = np.stack([S.coarse_step(U[: n + 1], sp, gr, pb, step_index=n) for n in range(lo, hi)])
    return lo, hi, f, g, list(sp.pcg_iterations)


def projections(states, seed=0, count=8):
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((states.shape[1], count))
    return states @ V


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--kmax", type=int, default=None)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--stride", type=int, default=None)
    a = ap.parse_args()
    i = a.config
    M, nt, m, alpha, T, tol = P.CONFIG_GRIDS[i]
    nt = a.nt or nt
    m = a.m or m
    k_max = a.kmax or nt + 1
    stride = a.stride or max(1, nt // 8)
    _init(i, M, nt, m, T)
    space, grids, prob = _W["space"], _W["grids"], _W["prob"]
    t0 = time.time()
    # parareal.py:91-155 (oracle.parareal.solve), with the parallel stage on processes
    u_curr = S.run_coarse(prob, space, grids)
    guard = DIVERGENCE_FACTOR * max(space.norm(u_curr[0]), 1.0)
    ni = space.size
    g_old = np.empty((nt, ni))
    f_old = np.empty((nt, ni))
    g_new = np.empty((nt, ni))
    diffs, pcg = [], []
    snaps = {}
    stop = "k_max"
    iterations = 0
    blocks = block_bounds(nt, min(a.procs, nt))
    with get_context("fork").Pool(len(blocks), initializer=_init, initargs=(i, M, nt, m, T)) as pool:
        for k in range(k_max):
            for lo, hi, f, g, its in pool.map(_block, [(u_curr, lo, hi) for lo, hi in blocks]):
                f_old[lo:hi] = f
                g_old[lo:hi] = g
                pcg.extend(its)
            u_next = np.empty_like(u_curr)
            u_next[0] = u_curr[0]
            for n in range(nt):
                g_new[n] = S.coarse_step(u_next[: n + 1], space, grids, prob, step_index=n)
                u_next[n + 1] = f_old[n] + (g_new[n] - g_old[n])
            if not np.isfinite(u_next).all():
                raise SystemExit(f"non-finite state at iteration {k}")
            if max(space.norm(u_next[n]) for n in range(nt + 1)) > guard:
                raise SystemExit(f"divergence guard at iteration {k}")
            diff = max(space.norm(u_next[n] - u_curr[n]) for n in range(nt + 1))
            diffs.append(diff)
            u_curr = u_next
            iterations = k + 1
            if k == 1:
                snaps[k + 1] = u_curr.copy()
            print(f"iteration {k + 1}: diff {diff:.3e} ({time.time() - t0:.0f} s, "
                  f"pcg mean {np.mean(pcg):.2f})", flush=True)
            if diff < tol:
                stop = "tol"
                break
    nodes = np.unique(np.r_[np.arange(0, nt + 1, stride), nt])
    suffix = "" if a.nt is None and a.m is None else f"_nt{nt}_m{m}"
    if a.kmax is not None:
        suffix += f"_k{a.kmax}"
    path = os.path.join(HERE, f"oracle_cfg{i}_2d{suffix}.npz")
    out = dict(nodes=nodes, states=u_curr[nodes], fine=f_old[nodes[nodes > 0] - 1],
               proj=projections(u_curr), norms=np.array([space.norm(v) for v in u_curr]),
               diffs=np.array(diffs), iterations=np.array(iterations), stop=np.array(stop),
               nt=np.array(nt), m=np.array(m), modes=np.array(M), pcg_mean=np.array(np.mean(pcg)))
    for k, v in snaps.items():
        out[f"states_k{k}"] = v[nodes]
    np.savez_compressed(path, **out)
    print(f"config {i} (P={nt}, m={m}, {M}^2 modes): {iterations} iterations ({stop}), "
          f"diffs {diffs}, {time.time() - t0:.0f} s -> {path}")


if __name__ == "__main__":
    main()
