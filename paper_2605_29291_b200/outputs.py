"""On-disk formats the reference's callers consume (SURVEY.md section 8(f),
row f2): the per-iteration trace CSV, the restart-log JSON and the run
summary JSON written by ``rapdb solve`` (cli.py:29-30, :49-61, :168-207).
Same columns, cell encodings (empty cell for a missing metric), key names
and atomic replace-on-write; the CLI verbs themselves are out of scope."""

from __future__ import annotations

import csv
import json
import os
import tempfile
import time
from typing import Iterable, Optional

TRACE_COLUMNS = ["iter", "tau", "sigma", "gamma", "evals", "kkt", "infeas",
                 "subopt", "gap_xi", "restart_flag"]      # cli.py:29-30


def _atomic_write(path: str, writer):
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, suffix=".tmp")
    try:
        with os.fdopen(fd, "w", newline="") as fh:
            writer(fh)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _cell(v):
    return "" if v is None else v


def write_trace_csv(path: str, trace: Iterable) -> None:
    """One row per accepted iteration; ``evals`` is the cumulative test count
    (cli.py:49-61)."""
    def emit(fh):
        w = csv.writer(fh)
        w.writerow(TRACE_COLUMNS)
        for rec in trace:
            w.writerow([rec.iter, rec.tau, rec.sigma, rec.gamma, rec.evals_total, _cell(rec.kkt),
                        _cell(rec.infeas), _cell(rec.subopt), _cell(rec.gap_xi), rec.restart_flag])
    _atomic_write(path, emit)


def write_json(path: str, obj) -> None:
    _atomic_write(path, lambda fh: json.dump(obj, fh, indent=2))


def restart_log_entries(restart_log) -> list:
    """cli.py:192-196."""
    return [{"outer": e.outer, "iteration": e.iteration, "trigger": e.trigger,
             "gap_new": e.gap_new, "gap_ref": e.gap_ref} for e in restart_log]


def run_summary(result, solver: str, wall_time_s: float) -> dict:
    """The summary dict of one rAPDB run (cli.py:176-185)."""
    return {
        "solver": solver,
        "iterations": result.iterations, "evals": result.evals,
        "restarts": len(result.restart_log),
        "converged": result.converged, "status": result.status,
        "wall_time_s": wall_time_s,
        "kkt": result.metrics.kkt_residual, "infeas": result.metrics.infeas,
        "f": result.metrics.f_value,
    }


def solve_and_write(inst, config, policy, solver: str, trace_csv: Optional[str] = None,
                    restart_json: Optional[str] = None, summary_json: Optional[str] = None,
                    **run_kw) -> dict:
    """``rapdb solve``'s output side around ``run_restarted``: returns the
    summary and writes whichever files are requested.  Exit-code convention
    of the reference: 0 if summary["converged"] else 2."""
    from .restarts import run_restarted
    start = time.monotonic()
    result = run_restarted(inst, config, policy, **run_kw)
    summary = run_summary(result, solver, time.monotonic() - start)
    if trace_csv:
        write_trace_csv(trace_csv, result.trace)
    if restart_json and result.restart_log:
        write_json(restart_json, restart_log_entries(result.restart_log))
    if summary_json:
        write_json(summary_json, summary)
    return summary
