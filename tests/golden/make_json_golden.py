"""Problem JSON written by the REAL reference (rapdb.problem.save) for its own
test instance, the eq-qp KAT and a small KML epigraph (zero Q_0 -> CSR) ->
tests/golden/problem_*.json.  Run in the build container."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from rapdb import generate, problem  # noqa: E402

problem.save(generate.random_qcqp(6, 2, seed=3), os.path.join(HERE, "problem_rq.json"))
eq = [a for a in generate.analytic_suite() if a.name == "eq-qp"][0].instance
problem.save(eq, os.path.join(HERE, "problem_eqqp.json"))
from paper_2605_29291_b200 import instances  # noqa: E402
from make_golden import ref_instance  # noqa: E402
problem.save(ref_instance(instances.kml_epigraph(N=12, d=3)), os.path.join(HERE, "problem_kml.json"))
print("ok")
