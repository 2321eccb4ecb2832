"""Trace CSV / summary / restart-log formats (outputs.py) against the
reference's own writer output (tests/golden/trace_ref.csv, made by
tests/golden/make_outputs_golden.py with rapdb.cli.write_trace_csv)."""

import json
import os

import pytest

from conftest import GOLDEN
from paper_2605_29291_b200 import outputs
from paper_2605_29291_b200.engine import TraceRecord
from paper_2605_29291_b200.restarts import RestartEvent


def records():
    out = []
    for k in range(1, 8):
        kkt = None if k % 3 else 10.0 ** (-k)
        out.append(TraceRecord(iter=k, tau_start=0.5 ** k, tau=0.5 ** k * 0.7, sigma=0.3 / k, gamma=1.0 + k / 7,
                               evals_iter=1 + (k % 2), evals_total=k + k // 2, kkt=kkt,
                               infeas=None if kkt is None else kkt / 3, subopt=None,
                               gap_xi=1e-9 * k if k == 4 else None, restart_flag=int(k == 5)))
    return out


def test_trace_csv_matches_reference_writer(tmp_path):
    p = tmp_path / "trace.csv"
    outputs.write_trace_csv(str(p), records())
    assert p.read_bytes() == open(os.path.join(GOLDEN, "trace_ref.csv"), "rb").read()


def test_restart_log_and_summary(tmp_path):
    log = [RestartEvent(outer=1, iteration=500, trigger="fixed"),
           RestartEvent(outer=2, iteration=700, trigger="adaptive", gap_new=1e-9, gap_ref=3e-9)]
    p = tmp_path / "r.json"
    outputs.write_json(str(p), outputs.restart_log_entries(log))
    got = json.loads(p.read_text())
    assert got == [{"outer": 1, "iteration": 500, "trigger": "fixed", "gap_new": None, "gap_ref": None},
                   {"outer": 2, "iteration": 700, "trigger": "adaptive", "gap_new": 1e-9, "gap_ref": 3e-9}]

    class M:
        kkt_residual, infeas, f_value = 1e-7, 2e-8, -3.0

    class Res:
        iterations, evals, restart_log, converged, status, metrics = 570, 595, log, True, "converged", M()

    s = outputs.run_summary(Res(), "rapdb-yx", 0.37)
    assert list(s) == ["solver", "iterations", "evals", "restarts", "converged", "status", "wall_time_s",
                       "kkt", "infeas", "f"]
    assert s["restarts"] == 2 and s["kkt"] == 1e-7


def test_atomic_write_leaves_no_temp_on_error(tmp_path):
    p = tmp_path / "x.json"
    with pytest.raises(TypeError):
        outputs.write_json(str(p), {"bad": object()})
    assert not p.exists() and not list(tmp_path.glob("*.tmp"))
