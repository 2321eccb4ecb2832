"""Trace CSV / restart-log JSON written by the REAL reference's writers
(cli.py:49-61) for a fixed synthetic trace -> tests/golden/trace_ref.csv.
Run in the build container (/root/reference present)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from rapdb import cli  # noqa: E402
from rapdb.engine import TraceRecord  # noqa: E402


def records(TR):
    out = []
    for k in range(1, 8):
        kkt = None if k % 3 else 10.0 ** (-k)
        out.append(TR(iter=k, tau_start=0.5 ** k, tau=0.5 ** k * 0.7, sigma=0.3 / k, gamma=1.0 + k / 7,
                      evals_iter=1 + (k % 2), evals_total=k + k // 2, kkt=kkt,
                      infeas=None if kkt is None else kkt / 3, subopt=None,
                      gap_xi=1e-9 * k if k == 4 else None, restart_flag=int(k == 5)))
    return out


if __name__ == "__main__":
    cli.write_trace_csv(os.path.join(HERE, "trace_ref.csv"), records(TraceRecord))
    print("wrote trace_ref.csv")
