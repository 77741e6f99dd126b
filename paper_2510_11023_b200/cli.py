"""Command-line front end on the device path.

Same subcommands, flags, ``[run]`` config-file format and CSV schemas as the
reference's ``parafrac`` CLI for the solver subset (``cli.py:193-257``), so a
GPU run and a CPU run of the same invocation produce side-by-side comparable
files:

* ``solve``    -> ``n,t,l2_norm,min,max`` per coarse node (``cli.py:193-205``)
* ``parareal`` -> ``k,max_diff[,err_vs_fine],wall_time_cumulative`` (``cli.py:208-240``)
* ``bench``    -> the 12 runtime/speedup/allocation columns (``cli.py:243-271``)

Two flags are added: ``--space {chebyshev,sine}`` and ``--dims`` (sine
only).  ``--n`` is the Chebyshev degree or the number of sine modes per axis.
Without ``--space`` the BASELINE problems ``cfg1``..``cfg5`` run in their sine
space and every other problem in the reference's Chebyshev space.  For a sine
space ``min``/``max`` are taken over the state vector as stored (coefficients),
exactly as the reference takes them over its stored nodal values.

``bounds`` and ``truncation`` (scalar analysis of the bound recurrences and of
the L1 operator, ``bounds.py``/``harness.py:126-227``) are not on the solver
path; they exit with status 2 and point at the reference CLI.

Exit codes follow ``cli.py:355-372``: 0 ok, 2 for argument/config/IO errors,
1 for solver errors (``ParafracError``).
"""

from __future__ import annotations

import argparse
import configparser
import dataclasses
import os
import sys
from dataclasses import dataclass

from .errors import ParafracError
from .harness import bench_sweep, make_operator
from .l1 import TimeGrids
from .problems import get_problem, registry_names
from .solver import parareal_solve, run_coarse, run_fine_sequential
from .spaces import l2_norm

__all__ = ["RunConfig", "build_parser", "emit_config", "main", "parse_config_text"]

SECTION = "run"
_FLOAT_FIELDS = ("alpha", "t_final", "tol")
_INT_FIELDS = ("nt", "m", "degree", "kmax", "threads", "reps", "dims")


@dataclass(frozen=True)
class RunConfig:
    """Effective settings of one invocation: defaults < config file < flags (``cli.py:31-70``)."""

    problem: str = "paper42"
    alpha: float | None = None
    t_final: float | None = None
    nt: int = 8
    m: int = 4
    degree: int | None = None
    tol: float = 1e-10
    kmax: int = 20
    threads: int | None = None
    out: str | None = None
    sweep: tuple = ()
    reference: bool = False
    solver: str = "fine"
    reps: int = 3
    space: str | None = None
    dims: int | None = None

    def validate(self):
        if self.nt < 1 or self.m < 1:
            raise ValueError("grid parameters nt, m must be >= 1")
        if self.degree is not None and self.degree < 2 and self.space != "sine":
            raise ValueError("degree must be >= 2")
        if not self.tol > 0:
            raise ValueError("tol must be positive")
        if self.kmax < 1:
            raise ValueError("kmax must be at least 1")
        if self.threads is not None and self.threads < 1:
            raise ValueError("threads must be at least 1")
        if self.reps < 1:
            raise ValueError("reps must be at least 1")
        if self.solver not in ("fine", "coarse"):
            raise ValueError("solver must be 'fine' or 'coarse'")
        if self.space not in (None, "chebyshev", "sine"):
            raise ValueError("space must be 'chebyshev' or 'sine'")
        if self.dims not in (None, 1, 2):
            raise ValueError("dims must be 1 or 2")
        if any(d < 1 for d in self.sweep):
            raise ValueError("sweep entries must be positive integers")
        return self


_FIELDS = {f.name: f for f in dataclasses.fields(RunConfig)}


def _coerce(name, text):
    text = text.strip()
    if name == "sweep":
        return tuple(int(tok) for tok in text.split(",") if tok.strip())
    if text == "":
        return None
    if name == "reference":
        return text.lower() in ("1", "true", "yes", "on")
    if name in _FLOAT_FIELDS:
        return float(text)
    if name in _INT_FIELDS:
        return int(text)
    return text


def parse_config_text(text):
    """``[run]`` section of ``key = value`` lines -> field overrides (``cli.py:96-112``)."""
    cp = configparser.ConfigParser()
    try:
        cp.read_string(text)
    except configparser.Error as exc:
        raise ValueError(f"malformed config: {exc}") from None
    if not cp.has_section(SECTION):
        raise ValueError(f"config must contain a [{SECTION}] section")
    out = {}
    for key, raw in cp.items(SECTION):
        if key == "n":  # the flag's name is accepted for the degree
            key = "degree"
        if key not in _FIELDS:
            raise ValueError(f"unknown config key {key!r}")
        out[key] = _coerce(key, raw)
    return out


def emit_config(cfg):
    """The effective config in the format ``parse_config_text`` reads back (round trip)."""
    lines = [f"[{SECTION}]"]
    for f in dataclasses.fields(RunConfig):
        v = getattr(cfg, f.name)
        if v is None:
            s = ""
        elif f.name == "sweep":
            s = ",".join(map(str, v))
        elif isinstance(v, bool):
            s = "true" if v else "false"
        elif isinstance(v, float):
            s = repr(v)
        else:
            s = str(v)
        lines.append(f"{f.name} = {s}")
    return "\n".join(lines) + "\n"


def _resolve(args):
    merged = {}
    if getattr(args, "config", None):
        with open(args.config, "r", encoding="utf-8") as fh:
            merged.update(parse_config_text(fh.read()))
    for name in _FIELDS:
        v = getattr(args, name, None)
        if v is not None:
            merged[name] = tuple(v) if name == "sweep" else v
    return RunConfig(**merged).validate()


def _cell(v):
    return f"{v:.16e}" if isinstance(v, float) else str(v)


def _write_csv(path, header, rows):
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(",".join(header) + "\n")
        for row in rows:
            fh.write(",".join(_cell(v) for v in row) + "\n")


def _threads(cfg):
    return cfg.threads if cfg.threads is not None else (os.cpu_count() or 1)


def _problem_space(cfg):
    problem = get_problem(cfg.problem, alpha=cfg.alpha, t_final=cfg.t_final)
    op = make_operator(problem, cfg.degree, cfg.space, cfg.dims)
    return problem, op, TimeGrids(problem.t_final, cfg.nt, cfg.m)


def cmd_solve(cfg):
    problem, op, grids = _problem_space(cfg)
    states = run_coarse(problem, op, grids) if cfg.solver == "coarse" else run_fine_sequential(problem, op, grids)[0]
    rows = [(n, n * grids.dT, l2_norm(op, states[n]), float(states[n].min()), float(states[n].max()))
            for n in range(grids.nt + 1)]
    out = cfg.out or "solve.csv"
    _write_csv(out, ("n", "t", "l2_norm", "min", "max"), rows)
    print(f"wrote {out} ({len(rows)} rows)", file=sys.stderr)
    return 0


def cmd_parareal(cfg):
    problem, op, grids = _problem_space(cfg)
    ref = ref_time = None
    if cfg.reference:
        ref, ref_time = run_fine_sequential(problem, op, grids)
    _, report = parareal_solve(problem, op, grids, tol=cfg.tol, k_max=cfg.kmax, threads=_threads(cfg),
                               reference=ref)
    report.wall_time_reference = ref_time
    header = ["k", "max_diff"] + (["err_vs_fine"] if cfg.reference else []) + ["wall_time_cumulative"]
    rows = []
    for k in range(1, report.iterations + 1):
        extra = [report.errors_vs_reference[k]] if cfg.reference else []
        rows.append([k, report.diffs[k - 1], *extra, report.iteration_times[k - 1]])
    out = cfg.out or "parareal.csv"
    _write_csv(out, header, rows)
    why = "tolerance" if report.stop_reason == "tol" else "iteration limit"
    print(f"stopped by {why} after {report.iterations} iterations (last diff {report.diffs[-1]:.3e}); "
          f"wrote {out}", file=sys.stderr)
    return 0


BENCH_HEADER = ("dof", "nt", "m", "degree", "threads", "wall_time_fine", "wall_time_parareal", "speedup",
                "iterations_used", "final_diff", "peak_alloc_bytes_fine_approx",
                "peak_alloc_bytes_parareal_approx")


def cmd_bench(cfg):
    if not cfg.sweep:
        raise ValueError("bench needs a nonempty --sweep list of dof values")
    recs = bench_sweep(cfg.problem, cfg.sweep, alpha=cfg.alpha, degree=cfg.degree, m=cfg.m, tol=cfg.tol,
                       k_max=cfg.kmax, threads=_threads(cfg), reps=cfg.reps, space=cfg.space, dims=cfg.dims)
    rows = [(r.dof, r.nt, r.m, r.degree, r.threads, r.wall_fine, r.wall_parareal, r.speedup, r.iterations,
             r.final_diff, r.peak_alloc_fine, r.peak_alloc_parareal) for r in recs]
    out = cfg.out or "bench.csv"
    _write_csv(out, BENCH_HEADER, rows)
    print(f"wrote {out} ({len(rows)} sweep points)", file=sys.stderr)
    return 0


def cmd_not_on_device(cfg):
    raise ValueError("this subcommand is scalar analysis outside the device solver path; "
                     "run it with the reference CLI (python -m parafrac.cli)")


COMMANDS = {"solve": cmd_solve, "parareal": cmd_parareal, "bench": cmd_bench,
            "bounds": cmd_not_on_device, "truncation": cmd_not_on_device}


def _sweep(text):
    try:
        return tuple(int(tok) for tok in text.split(",") if tok.strip())
    except ValueError:
        raise argparse.ArgumentTypeError(f"not a comma list of integers: {text!r}") from None


def _common(p, grid=True):
    p.add_argument("--config", help="key = value config file ([run] section)")
    p.add_argument("--out", help="output CSV path")
    if not grid:
        return
    p.add_argument("--problem", choices=registry_names(), help="builtin problem")
    p.add_argument("--alpha", type=float, help="fractional order in (0, 1]")
    p.add_argument("--nt", type=int, help="coarse intervals (parareal slices)")
    p.add_argument("--m", type=int, help="fine steps per coarse interval")
    p.add_argument("--n", type=int, dest="degree", help="Chebyshev degree / sine modes per axis")
    p.add_argument("--tol", type=float, help="parareal stopping tolerance")
    p.add_argument("--kmax", type=int, help="parareal iteration cap")
    p.add_argument("--threads", type=int, help="accepted for compatibility (the device batches all slices)")
    p.add_argument("--space", choices=("chebyshev", "sine"), help="spatial discretisation")
    p.add_argument("--dims", type=int, choices=(1, 2), help="sine space dimension")


def build_parser():
    parser = argparse.ArgumentParser(prog="paper_2510_11023_b200",
                                     description="B200 parareal-L1-spectral solver (parafrac-compatible CLI)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="one solver, coarse-node trajectory CSV")
    _common(p)
    p.add_argument("--solver", choices=("fine", "coarse"), help="which propagator to run")
    p = sub.add_parser("parareal", help="parareal iteration, per-iteration CSV")
    _common(p)
    p.add_argument("--reference", action="store_true", default=None,
                   help="also run the serial fine solver and report errors against it")
    p = sub.add_parser("bench", help="fine vs parareal timing over a dof sweep")
    _common(p)
    p.add_argument("--sweep", type=_sweep, help="comma list of dof values")
    p.add_argument("--reps", type=int, help="timing repetitions (the minimum is reported)")
    for name in ("bounds", "truncation"):
        p = sub.add_parser(name, help="not on the device path (use the reference CLI)")
        _common(p, grid=False)
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        cfg = _resolve(args)
        print(f"paper_2510_11023_b200 {args.command}: problem={cfg.problem} threads={_threads(cfg)}",
              file=sys.stderr)
        return COMMANDS[args.command](cfg)
    except (ValueError, OverflowError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except ParafracError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
