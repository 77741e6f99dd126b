"""The parafrac-compatible CLI and bench harness.

CPU tests cover the config-file format, validation and exit codes (the
reference's ``test_cli.py`` contract); the ``gpu`` tests run the subcommands
through the device path and check the CSV contents against the oracle."""

import csv
import math

import numpy as np
import pytest

import oracle
from oracle import problems as OP
from paper_2510_11023_b200 import cli, harness
import paper_2510_11023_b200 as pfb


def _rows(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


# ------------------------------------------------------------------ CPU: config, validation, exit codes
def test_config_round_trip():
    cfg = cli.RunConfig(problem="cfg1", alpha=0.5, nt=4, m=8, degree=16, sweep=(64, 128), reference=True,
                        space="sine", dims=1, threads=2)
    back = cli.RunConfig(**cli.parse_config_text(cli.emit_config(cfg)))
    assert back == cfg


def test_config_accepts_flag_name_for_degree():
    assert cli.parse_config_text("[run]\nn = 12\n") == {"degree": 12}


@pytest.mark.parametrize("text", ["nt = 3\n", "[run]\nbogus = 1\n", "[run\nnt=3"])
def test_config_errors(text):
    with pytest.raises(ValueError):
        cli.parse_config_text(text)


@pytest.mark.parametrize("argv", [
    ["solve", "--nt", "0"],
    ["parareal", "--tol", "0"],
    ["parareal", "--kmax", "0"],
    ["bench", "--m", "4"],                      # empty sweep
    ["solve", "--threads", "0"],
    ["bounds"], ["truncation"],                 # not on the device path
])
def test_argument_errors_exit_2(argv, capsys):
    assert cli.main(argv) == 2
    assert "error:" in capsys.readouterr().err


def test_flags_override_config_file(tmp_path):
    path = tmp_path / "run.ini"
    path.write_text("[run]\nproblem = cfg2\nnt = 6\nm = 5\n")
    args = cli.build_parser().parse_args(["parareal", "--config", str(path), "--m", "9"])
    cfg = cli._resolve(args)
    assert (cfg.problem, cfg.nt, cfg.m) == ("cfg2", 6, 9)


def test_operator_choice():
    p42 = pfb.get_problem("paper42")
    assert isinstance(harness.make_operator(p42), pfb.ChebyshevOperator)
    assert harness.make_operator(p42).degree == 16
    op = harness.make_operator(pfb.get_problem("cfg4"))
    assert isinstance(op, pfb.SineOperator) and (op.modes, op.dims) == (128, 2)
    op = harness.make_operator(pfb.get_problem("cfg1"), degree=16)
    assert (op.modes, op.dims) == (16, 1)
    with pytest.raises(ValueError):
        harness.make_operator(p42, space="fourier")


# ------------------------------------------------------------------ GPU: subcommands through the device path
@pytest.mark.gpu
def test_solve_csv_matches_oracle(tmp_path):
    out = tmp_path / "solve.csv"
    assert cli.main(["solve", "--problem", "paper42", "--n", "8", "--nt", "4", "--m", "4", "--out", str(out)]) == 0
    rows = _rows(out)
    assert rows[0] == ["n", "t", "l2_norm", "min", "max"]
    sp = oracle.build_operator(8, 0.0, 1.0)
    states, _ = oracle.run_fine_sequential(OP.paper42(), sp, oracle.TimeGrids(1.0, 4, 4))
    assert len(rows) == 1 + 5
    for n, row in enumerate(rows[1:]):
        assert int(row[0]) == n and math.isclose(float(row[1]), n * 0.25)
        assert abs(float(row[2]) - sp.norm(states[n])) <= 1e-12 * max(1.0, sp.norm(states[n]))
        assert abs(float(row[3]) - states[n].min()) <= 1e-12 and abs(float(row[4]) - states[n].max()) <= 1e-12
        assert "e" in row[2]  # %.16e cells, as the reference writes them


@pytest.mark.gpu
def test_parareal_csv_config1(tmp_path):
    out = tmp_path / "parareal.csv"
    argv = ["parareal", "--problem", "cfg1", "--nt", "8", "--m", "64", "--tol", "1e-12", "--reference",
            "--out", str(out)]
    assert cli.main(argv) == 0
    rows = _rows(out)
    assert rows[0] == ["k", "max_diff", "err_vs_fine", "wall_time_cumulative"]
    sp, g = oracle.Sine1D(32), oracle.TimeGrids(1.0, 8, 64)
    ref, _ = oracle.run_fine_sequential(OP.config(1), sp, g)
    o_it, o_rep = oracle.parareal_solve(OP.config(1), sp, g, tol=1e-12, reference=ref)
    assert len(rows) - 1 == o_rep.iterations == 9
    diffs = np.array([float(r[1]) for r in rows[1:]])
    np.testing.assert_allclose(diffs[:-2], np.array(o_rep.diffs)[:-2], rtol=1e-3)
    times = [float(r[3]) for r in rows[1:]]
    assert all(b >= a for a, b in zip(times, times[1:]))
    # error of each iterate against the serial fine solution (the parareal fixed
    # point differs from it by the coarse-compressed history, ~1e-3 here)
    errs = np.array([float(r[2]) for r in rows[1:]])
    np.testing.assert_allclose(errs, np.array(o_rep.errors_vs_reference[1:]), rtol=1e-8)


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    out = tmp_path / "bench.csv"
    argv = ["bench", "--problem", "cfg1", "--n", "16", "--m", "16", "--sweep", "64,128", "--reps", "1",
            "--tol", "1e-12", "--out", str(out)]
    assert cli.main(argv) == 0
    rows = _rows(out)
    assert tuple(rows[0]) == cli.BENCH_HEADER
    assert [int(r[0]) for r in rows[1:]] == [64, 128]
    assert [int(r[1]) for r in rows[1:]] == [4, 8]
    for r in rows[1:]:
        assert float(r[5]) > 0 and float(r[6]) > 0 and float(r[9]) < 1e-12
