timeout 600 python tools/measure_configs.py C1 20000 mono adaptive > gpurun_out/m_c1_ada.json 2>gpurun_out/e1; cut -c1-420 gpurun_out/m_c1_ada.json; echo
timeout 600 python tools/measure_configs.py C1 20000 nm adaptive > gpurun_out/m_c1_nmada.json 2>gpurun_out/e2; cut -c1-420 gpurun_out/m_c1_nmada.json; echo
python - <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
arr = instances.config_instance("C1")
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
for mode, nm in (("xy", False), ("xy", True)):
    t0 = time.perf_counter()
    res = R.run_restarted(inst, R.SolverConfig(mode=mode, nonmonotone=nm), R.FixedRestart(500), budget=20000, criteria=crit)
    torch.cuda.synchronize()
    print(mode, "nm" if nm else "mono", res.iterations, res.evals, res.converged, f"{time.perf_counter()-t0:.3f}s", res.metrics.kkt_residual)
PY
