import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
t=time.time(); arr = instances.config_instance(sys.argv[1] if len(sys.argv)>1 else "C1"); print("gen", time.time()-t, flush=True)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
t=time.time(); d = inst.device_data("cuda:0"); torch.cuda.synchronize(); print("upload", time.time()-t, flush=True)
ev = inst._evaluator()
x = torch.from_numpy(np.random.default_rng(0).uniform(-1,1,arr.n)).cuda()
for reps in (1, 20):
    u, g, ms = ev.ctx.probe_sweep(x, reps=reps)
    print("probe reps", reps, "ms/sweep (launch avg)", ms, "GB/s", (arr.m+1)*arr.n*arr.n*8/ms/1e6, flush=True)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
for nm, pol in ((False, R.FixedRestart(500)), (True, R.FixedRestart(500)), (True, R.NoRestart()), (False, R.NoRestart())):
    torch.cuda.synchronize(); t = time.time()
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=nm), pol, budget=int(sys.argv[2]) if len(sys.argv)>2 else 20000, criteria=crit)
    dt = time.time() - t
    st = res.device_stats
    print(f"nm={nm} pol={pol} iters={res.iterations} evals={res.evals} conv={res.converged} wall={dt:.2f}s it/s={res.iterations/dt:.1f} kkt={res.metrics.kkt_residual:.2e} f={res.metrics.f_value:.8e} sweep_ms={st['sweep_ns']/st['sweeps']/1e6:.4f} sweepGBs={(arr.m+1)*arr.n*arr.n*8/(st['sweep_ns']/st['sweeps']):.1f}", flush=True)
    kk = [(t.iter, t.kkt) for t in res.trace if t.kkt is not None]
    print("  kkt trail", [(a, f"{b:.1e}") for a, b in kk[::max(1,len(kk)//12)]], flush=True)
