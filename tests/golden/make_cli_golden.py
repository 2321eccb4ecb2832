"""Outputs of the REAL reference CLI (`rapdb solve` / `rapdb gap`,
cli.py:188-271) on the committed problem JSON files -> tests/golden/cli/.
Run in the build container (/root/reference present); the GPU test
tests/test_gpu_cli.py runs paper_2605_29291_b200.cli with the same argv and
compares files and exit codes."""
import contextlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")
from rapdb import cli  # noqa: E402

# (case name, problem file, extra argv) -- shared with tests/test_gpu_cli.py
CASES = [
    ("rq_yx", "problem_rq.json", ["--solver", "rapdb-yx"]),
    ("rq_yx_ada", "problem_rq.json", ["--solver", "rapdb-yx-ada"]),
    ("rq_xy_nm", "problem_rq.json", ["--solver", "rapdb-xy", "--nonmonotone", "--restart", "fixed:200", "--budget", "1500"]),
    ("rq_apdb_ball", "problem_rq.json", ["--solver", "apdb-yx", "--dual-bound", "50", "--budget", "400"]),
    ("kml_yx", "problem_kml.json", ["--solver", "rapdb-yx", "--eps", "1e-6"]),
    ("eq_yx", "problem_eqqp.json", ["--solver", "rapdb-yx", "--budget", "3000"]),
    ("rq_egm", "problem_rq.json", ["--solver", "egm", "--stepsize", "0.01", "--budget", "300"]),
    ("rq_short", "problem_rq.json", ["--solver", "rapdb-yx", "--budget", "30"]),
]

GAP_CASES = [
    ("rq_gap0", "problem_rq.json", []),
    ("rq_gap_xi", "problem_rq.json", ["--xi", "0.5"]),
    ("eq_gap0", "problem_eqqp.json", []),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    codes = {}
    for name, prob, extra in CASES:
        argv = ["solve", "--problem", os.path.join(HERE, prob), *extra,
                "--out", os.path.join(OUT, name + ".csv"), "--summary", os.path.join(OUT, name + ".json"),
                "--restart-log", os.path.join(OUT, name + "_restarts.json")]
        codes[name] = cli.main(argv)
        print(name, codes[name], flush=True)
    gaps = {}
    for name, prob, extra in GAP_CASES:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = cli.main(["gap", "--problem", os.path.join(HERE, prob), *extra])
        gaps[name] = {"argv": [prob, *extra], "exit": code, "out": json.loads(buf.getvalue())}
        print(name, code, flush=True)
    with open(os.path.join(OUT, "cases.json"), "w") as fh:
        json.dump({"solve": [{"name": n, "problem": p, "argv": e, "exit": codes[n]} for n, p, e in CASES],
                   "gap": gaps}, fh, indent=1)


if __name__ == "__main__":
    main()
