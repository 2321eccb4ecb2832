"""The ``solve`` / ``gap`` verbs (paper_2605_29291_b200.cli) against the REAL
reference CLI's files and exit codes (tests/golden/cli, made by
tests/golden/make_cli_golden.py with rapdb.cli.main on the same argv).

CPU tests: argument handling, restart specs, solver-name mapping, config
precedence and the exit-1 paths (no device work).  GPU tests: every golden
case end to end through the device solver -- same exit code, summary keys and
counts, trace rows (iter / evals / restart_flag exact; tau, sigma, gamma to
1e-12 relative; metric cells present in the same rows, values to 1e-6),
restart log and smoothed-gap output."""

import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_29291_b200 import cli, restarts

CLI_DIR = os.path.join(GOLDEN, "cli")
CASES = json.load(open(os.path.join(CLI_DIR, "cases.json")))


def _args(argv):
    return cli.merge_config(cli.build_parser().parse_args(argv))


# ---------------------------------------------------------------- CPU side

def test_restart_specs_follow_the_mode():
    assert isinstance(cli.parse_restart(None, "yx"), restarts.NoRestart)
    assert isinstance(cli.parse_restart("none", "yx"), restarts.NoRestart)
    assert cli.parse_restart("fixed", "yx").period == 500
    assert cli.parse_restart("fixed:200", "xy").period == 200
    a = cli.parse_restart("adaptive", "yx")
    assert (a.xi, a.q, a.warmup, a.check_period) == (0.04, 0.5, 50, 200)
    a = cli.parse_restart("adaptive:0.1,0.25", "xy")
    assert (a.xi, a.q, a.warmup, a.check_period) == (0.1, 0.25, 100, 500)
    with pytest.raises(cli.InputError):
        cli.parse_restart("sometimes", "yx")


def test_solver_names_map_to_config_and_policy():
    base = ["solve", "--problem", "p.json", "--solver", "x"]
    cfg, pol = cli.solver_setup("rapdb-xy", _args(base))
    assert cfg.mode == "xy" and isinstance(pol, restarts.FixedRestart) and pol.period == 500
    cfg, pol = cli.solver_setup("apdb-yx", _args(base + ["--restart", "fixed:9"]))
    assert cfg.mode == "yx" and isinstance(pol, restarts.NoRestart)
    cfg, pol = cli.solver_setup("rapdb-yx-ada", _args(base + ["--nonmonotone", "--dual-bound", "3"]))
    assert cfg.nonmonotone and isinstance(pol, restarts.AdaptiveRestart) and cfg.dual_ball.radius == 3.0
    assert cli.solver_setup("egm", _args(base)) == (None, None)
    with pytest.raises(cli.InputError):
        cli.solver_setup("newton", _args(base))


def test_config_file_fills_only_unset_flags(tmp_path):
    cfgp = tmp_path / "c.json"
    cfgp.write_text(json.dumps({"nonmonotone": True, "restart": "fixed:7", "dual-bound": 4.0}))
    a = _args(["solve", "--problem", "p", "--solver", "rapdb-yx", "--restart", "none", "--config", str(cfgp)])
    assert a.nonmonotone is True and a.restart == "none" and a.dual_bound == 4.0
    a = _args(["solve", "--problem", "p", "--solver", "rapdb-yx"])
    assert a.nonmonotone is False


def test_bad_input_exits_1(tmp_path, capsys):
    rq = os.path.join(GOLDEN, "problem_rq.json")
    assert cli.main(["solve", "--problem", rq, "--solver", "newton"]) == 1
    assert cli.main(["solve", "--problem", str(tmp_path / "missing.json"), "--solver", "rapdb-yx"]) == 1
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["solve", "--problem", str(bad), "--solver", "rapdb-yx"]) == 1
    assert cli.main(["gen", "--family", "random-qcqp", "--out", str(tmp_path / "o.json")]) == 1
    assert cli.main(["bound", "--problem", rq]) == 1
    assert "error:" in capsys.readouterr().err


def test_golden_cases_are_complete():
    names = {c["name"] for c in CASES["solve"]}
    for n in names:
        assert os.path.exists(os.path.join(CLI_DIR, n + ".json"))
        assert os.path.exists(os.path.join(CLI_DIR, n + ".csv"))
    assert {c["exit"] for c in CASES["solve"]} == {0, 2}


# ---------------------------------------------------------------- GPU side

def _rows(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


def _close(a, b, rtol, atol=0.0):
    return abs(a - b) <= atol + rtol * max(abs(a), abs(b))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES["solve"], ids=lambda c: c["name"])
def test_solve_matches_reference_cli(case, tmp_path):
    name = case["name"]
    out = {k: str(tmp_path / (name + suf)) for k, suf in (("csv", ".csv"), ("sum", ".json"), ("log", "_r.json"))}
    code = cli.main(["solve", "--problem", os.path.join(GOLDEN, case["problem"]), *case["argv"],
                     "--out", out["csv"], "--summary", out["sum"], "--restart-log", out["log"]])
    assert code == case["exit"]
    ref = json.load(open(os.path.join(CLI_DIR, name + ".json")))
    got = json.load(open(out["sum"]))
    assert list(got) == list(ref)
    nm = "--nonmonotone" in case["argv"]
    for k in ("solver", "iterations", "converged", "status", "restarts", "diverged", "stepsize"):
        if k in ref:
            assert got[k] == ref[k], k
    if nm:   # non-monotone accept decisions are rounding-sensitive
        assert abs(got["evals"] - ref["evals"]) <= 0.02 * ref["evals"]
    else:
        assert got["evals"] == ref["evals"]
    for k in ("kkt", "infeas", "f"):
        assert _close(got[k], ref[k], 1e-6, 1e-9), (k, got[k], ref[k])

    ref_rows = _rows(os.path.join(CLI_DIR, name + ".csv"))
    got_rows = _rows(out["csv"])
    assert got_rows[0] == ref_rows[0]
    assert len(got_rows) == len(ref_rows)
    cols = ref_rows[0]
    exact = [cols.index(c) for c in ("iter", "evals", "restart_flag")]
    steps = [cols.index(c) for c in ("tau", "sigma", "gamma")]
    metric = [cols.index(c) for c in ("kkt", "infeas", "subopt", "gap_xi")]
    for r, (g, e) in enumerate(zip(got_rows[1:], ref_rows[1:])):
        if nm and r >= 200:
            break
        for j in exact:
            assert g[j] == e[j], (r, cols[j])
        for j in steps:
            assert _close(float(g[j]), float(e[j]), 1e-12), (r, cols[j], g[j], e[j])
        for j in metric:
            assert (g[j] == "") == (e[j] == ""), (r, cols[j])
            if e[j] != "":
                assert _close(float(g[j]), float(e[j]), 1e-6, 1e-10), (r, cols[j], g[j], e[j])

    ref_log = os.path.join(CLI_DIR, name + "_restarts.json")
    assert os.path.exists(out["log"]) == os.path.exists(ref_log)
    if os.path.exists(ref_log):
        a, b = json.load(open(out["log"])), json.load(open(ref_log))
        if not nm:
            assert len(a) == len(b)
        for x, y in zip(a, b):
            assert (x["outer"], x["iteration"], x["trigger"]) == (y["outer"], y["iteration"], y["trigger"])
            for k in ("gap_new", "gap_ref"):
                assert (x[k] is None) == (y[k] is None)
                if y[k] is not None:
                    assert _close(x[k], y[k], 1e-6, 1e-12), (k, x[k], y[k])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES["gap"]))
def test_gap_matches_reference_cli(name, capsys):
    case = CASES["gap"][name]
    prob, *extra = case["argv"]
    assert cli.main(["gap", "--problem", os.path.join(GOLDEN, prob), *extra]) == case["exit"]
    got = json.loads(capsys.readouterr().out)
    ref = case["out"]
    assert list(got) == list(ref)
    assert got["xi"] == ref["xi"] and got["reliable"] == ref["reliable"]
    assert np.isclose(got["gap"], ref["gap"], rtol=1e-8, atol=1e-12)
    assert abs(got["subsolver_iterations"] - ref["subsolver_iterations"]) <= 10


def test_module_entry_point_exit_code():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "paper_2605_29291_b200", "solve", "--problem",
                        os.path.join(GOLDEN, "problem_rq.json"), "--solver", "newton"],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 1 and "unknown solver" in r.stderr


@pytest.mark.gpu
def test_solve_binary_stack_matches_json(tmp_path):
    """--problem as the binary stack (problem.save_stack, .npz): the same run
    as from the reference's problem JSON."""
    from paper_2605_29291_b200 import problem
    src = os.path.join(GOLDEN, "problem_rq.json")
    npz = str(tmp_path / "rq.npz")
    problem.save_stack(problem.load(src), npz)
    outs = {}
    for name, path in (("json", src), ("npz", npz)):
        s = str(tmp_path / (name + ".json"))
        c = str(tmp_path / (name + ".csv"))
        assert cli.main(["solve", "--problem", path, "--solver", "rapdb-yx", "--summary", s, "--out", c]) == 0
        outs[name] = (json.load(open(s)), open(c).read())
    a, b = outs["json"], outs["npz"]
    assert a[1] == b[1]
    for k in ("iterations", "evals", "converged", "kkt", "infeas", "f"):
        assert a[0][k] == b[0][k]


@pytest.mark.gpu
def test_gap_at_a_given_point(tmp_path, capsys):
    """gap --point {x, v, lam}: the device smoothed gap at that point agrees
    with the oracle's restatement of diagnostics.smoothed_gap."""
    from oracle import rapdb_oracle as O
    from paper_2605_29291_b200 import problem
    src = os.path.join(GOLDEN, "problem_rq.json")
    inst = problem.load(src)
    rng = np.random.default_rng(5)
    x = rng.uniform(-0.5, 0.5, inst.n)
    lam = rng.uniform(0.0, 1.0, inst.m)
    pt = tmp_path / "pt.json"
    pt.write_text(json.dumps({"x": x.tolist(), "lam": lam.tolist()}))
    assert cli.main(["gap", "--problem", src, "--point", str(pt), "--xi", "0.1"]) == 0
    got = json.loads(capsys.readouterr().out)
    P = O.Problem(list(np.asarray(inst.Q)), list(np.asarray(inst.q)), inst.r, inst.A, inst.b,
                  inst.primal_set.lower, inst.primal_set.upper, inst.mu)
    ref_gap = O.smoothed_gap(P, x, np.zeros(inst.p), lam, 0.1)[0]
    assert np.isclose(got["gap"], ref_gap, rtol=1e-8, atol=1e-12)
