"""Benchmark: rAPDB on BASELINE.json config 1 (dense QCQP n=2000, m=200) on B200.

A "step" is one full drop-in solve, ``run_restarted`` of C1 to the conic
KKT / feasibility tolerance 1e-6 (``metrics_every=10``) with the reference
CLI's rapdb-yx policy (``FixedRestart(500)``, cli.py:90-107) and monotone
backtracking (the variant that converges on C1; the non-monotone variant is
timed on a fixed 1000-iteration budget and reported under ``nonmonotone``).

* ``value``        accepted iterations / s, Q stack resident in HBM.  N ranks
                   (torchrun): the constraints are sharded over the GPUs and each
                   trial all-reduces one n-vector and one (m+1)-vector over NCCL
                   (``scaling: strong``, one solve); ``--replicas`` runs
                   independent replicas instead (``scaling: weak``).
* ``ms_per_step``  = time-to-1e-6-KKT of one solve.
* ``e2e``          the same solve through the public API with the instance on
                   the HOST: pinned H2D of the 6.4 GB Q stack + vectors, solve,
                   D2H of solution/average/trace/metrics, all inside the timing.
* ``roofline``     the solver kernel: algorithmic Q bytes streamed (sweeps x
                   (m+1) n^2 8 B) / CUDA-event duration of its launches.
* ``cpu_baseline`` the CPU oracle (numpy restatement of the reference, same
                   arithmetic and matvec count) on a bounded sample of C1 iterations.

``--impl reference`` times that CPU restatement alone (the reference is pure
Python: nothing is compiled into oracle/_ref).  Inputs (6.4 GB) exceed the
126 MB L2, so no L2 flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rAPDB iters/s & time-to-1e-6 KKT; Q-sweep HBM GB/s vs B200 peak"
UNIT = "iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--replicas", action="store_true",
                    help="with N>1: independent replicas instead of constraint sharding")
    ap.add_argument("--shard", action="store_true",
                    help="force the constraint-sharded (NCCL exchange) path even with one rank")
    ap.add_argument("--p2p", action="store_true",
                    help="sharded runs exchange in-kernel over NVLink peer memory instead of NCCL")
    ap.add_argument("--cpu-sample-iters", type=int, default=24,
                    help="accepted C1 iterations per CPU sample (~0.25 s each on 16 cores)")
    ap.add_argument("--skip-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


_RESULT_OUT = None


def emit(out):
    """The one JSON result line, on the original stdout (library chatter such
    as NCCL's version banner is routed to stderr)."""
    stream = _RESULT_OUT if _RESULT_OUT is not None else sys.stdout
    stream.write(json.dumps(out) + "\n")
    stream.flush()


def _claim_stdout():
    global _RESULT_OUT
    sys.stdout.flush()
    _RESULT_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas"]
                   or [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(arr, iters, warm_iters=1):
    """CPU oracle: `iters` accepted mono-yx iterations after `warm_iters` (bounded sample)."""
    from oracle import rapdb_oracle as O
    P = O.Problem.from_arrays(arr)
    opt = O.Options(mode="yx", nonmonotone=False)
    eng = O.Engine(P, opt, *O.initial_point(P))
    for _ in range(warm_iters):
        eng.step()
    t0 = time.perf_counter()
    for _ in range(iters):
        eng.step()
    dt = time.perf_counter() - t0
    return iters / dt, dt, eng


def config_block(arr, name, policy, extra=None):
    d = {"workload": f"{name}: dense convex QCQP n={arr.n}, m={arr.m}, B_i rank {arr.meta.get('rank')}, "
                     f"Q stack {(arr.m + 1) * arr.n * arr.n * 8 / 1e9:.3f} GB fp64",
         "n": arr.n, "m": arr.m, "policy": policy, "tolerance": "conic KKT<=1e-6 and infeas<=1e-6",
         "metrics_every": 10, "seed": 0, "inputs_larger_than_l2": True, "l2_flush": False}
    if extra:
        d.update(extra)
    return d


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2605_29291_b200 import instances
    if args.config == "C2":
        emit({"impl": "reference", "unavailable": "C2's 69 GB dense stack does not fit the CPU reference's host"})
        return
    arr = instances.config_instance(args.config)
    from oracle import rapdb_oracle as O
    P = O.Problem.from_arrays(arr)
    eng = O.Engine(P, O.Options(mode="yx", nonmonotone=False), *O.initial_point(P))
    eng.step()                      # the first iteration backtracks from tau_bar (excluded)
    for _ in range(args.warmup):
        eng.step()
    per_step = max(1, args.cpu_sample_iters)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(per_step):
            eng.step()
    dt = time.perf_counter() - t0
    iters = args.steps * per_step
    v = iters / dt
    cores = blas_threads()
    sample = (f"{args.steps} steps x {per_step} accepted mono-yx iterations of {args.config} "
              f"(after {1 + args.warmup} warm-up iterations), numpy/OpenBLAS restatement of the reference")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded CounterRng, BASELINE config 1 shapes)",
           "config": config_block(arr, args.config, "yx monotone, per-step sample of accepted iterations"),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def main():
    args = parse()
    _claim_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    ws, rank, local = dist_env()
    sharded = (ws > 1 and not args.replicas) or args.shard
    os.environ.setdefault("NCCL_DEBUG", "WARN")     # keep stdout to the one JSON line
    if ws > 1 or args.shard:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if not dist.is_initialized():
            if ws == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29511")
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl")
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_2605_29291_b200 as R
    from paper_2605_29291_b200 import _capi, instances
    from paper_2605_29291_b200.sharding import nccl_shard

    device_generated = args.config == "C2"
    if device_generated:
        # the C2 host instance needs ~69 GB of host RAM and minutes of BLAS:
        # generate and pack the stack on the device (same distribution)
        inst = R.DeviceDenseInstance(4096, 512, 256, seed=0, name="C2 (device-generated)")
        arr = inst
    else:
        arr = instances.config_instance(args.config)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
    cfg = R.SolverConfig(mode="yx", nonmonotone=False)
    pol = R.FixedRestart(500)
    crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    shard = None
    if sharded:
        shard = nccl_shard(inst)
        shard.force_split = True
        shard.p2p = bool(args.p2p)
    krange = None if shard is None else (shard.k0, shard.k1)

    def solve(c=cfg, budget=50_000, criteria=crit):
        return R.run_restarted(inst, c, pol, budget=budget, criteria=criteria, metrics_every=10, device=dev,
                               shard=shard)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    inst.device_data(dev, krange=krange)
    for _ in range(args.warmup):
        solve()

    # ---- device-resident timed region -----------------------------------
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    launches0 = _capi.launch_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    results = [solve() for _ in range(args.steps)]
    ev1.record()
    barrier()
    launches = _capi.launch_count() - launches0
    clk = clocks.stop()
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    iters_local = sum(r.iterations for r in results)
    # sharded: every rank runs the same solve (strong scaling); replicas: sum
    iters_all = iters_local if sharded else sum_over_ranks(iters_local)
    value = iters_all / (t_ms / 1e3)
    conv = all(r.converged for r in results)
    st = results[-1].device_stats
    sweep_bytes = st["sweep_bytes"]
    layout = os.environ.get("RAPDB_LAYOUT", "packed")
    dense_bytes = (arr.m + 1 if shard is None else shard.k1 - shard.k0) * arr.n * arr.n * 8
    kern_ms = sum(r.device_stats["kernel_ms"] for r in results)
    sweeps = sum(r.device_stats["sweeps"] for r in results)
    sweep_ns = sum(r.device_stats["sweep_ns"] for r in results)
    achieved = sweeps * sweep_bytes / (kern_ms / 1e3) / 1e9
    sweep_phase_gbs = sweeps * sweep_bytes / sweep_ns
    peak, peak_src = measured_peak()

    # standalone sweep launch (one kernel launch = one fused sweep), CUDA events
    probe_ms = None
    if shard is None:
        ev = inst._evaluator()
        xprobe = torch.from_numpy(np.asarray(results[-1].solution.x)).to(dev)
        ev.ctx.probe_sweep(xprobe, reps=1)
        _, _, probe_ms = ev.ctx.probe_sweep(xprobe, reps=10)

    # ---- e2e through the public API with host-resident inputs -----------
    if device_generated:
        e2e_block = {"unavailable": "device-generated instance: its inputs never exist on the host"}
    else:
        e2e_block = None
        inst.pin_host()
        inst.drop_device_data()
    torch.cuda.synchronize()
    nloc = arr.m + 1 if shard is None else shard.k1 - shard.k0
    if layout == "packed" and os.environ.get("RAPDB_PACK_STAGED", "0") != "1":
        # packed straight from page-locked host memory: only the stored upper
        # block triangle crosses PCIe
        from paper_2605_29291_b200.problem import packed_source_elements
        q_bytes = nloc * packed_source_elements(arr.n) * 8
    else:
        q_bytes = nloc * arr.n * arr.n * 8
    h2d = q_bytes + inst.q.nbytes + inst.r.nbytes + 2 * arr.n * 8 + inst.A.nbytes + inst.b.nbytes
    e2e_iters, e2e_s, d2h = 0, 0.0, 0
    for _ in range(0 if device_generated else args.steps):
        inst.drop_device_data()
        barrier()
        t0 = time.perf_counter()
        r = solve()
        sol = (r.solution.x, r.average.x)
        barrier()
        e2e_s += time.perf_counter() - t0
        e2e_iters += r.iterations
        d2h = (2 * (arr.n + arr.m + arr.p) * 8 + r.device_stats["run_launches"] * 0
               + r.iterations * 11 * 8 + 8 * 8)
    e2e_s = max_over_ranks(e2e_s)
    e2e_value = (e2e_iters if sharded else sum_over_ranks(e2e_iters)) / e2e_s if e2e_s > 0 else None

    # non-monotone variant: fixed 1000-iteration budget (it/s only)
    inst.device_data(dev, krange=krange)
    nm_cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    torch.cuda.synchronize()
    tn = time.perf_counter()
    rnm = solve(c=nm_cfg, budget=1000)
    torch.cuda.synchronize()
    tn = time.perf_counter() - tn

    out = None
    if rank == 0:
        cpu = None
        if not args.skip_cpu and ws == 1 and not device_generated:
            v_cpu, dt_cpu, _ = oracle_sample(arr, args.cpu_sample_iters)
            cpu = {"value": v_cpu, "unit": UNIT, "cores": blas_threads(), "kind": "port",
                   "sample": f"{args.cpu_sample_iters} accepted mono-yx iterations of C1 after the first "
                             f"(backtracking) iteration, numpy/OpenBLAS restatement of the reference "
                             f"(oracle/rapdb_oracle.py), {dt_cpu:.1f} s",
                   "extrapolated_time_to_kkt_s": results[-1].iterations / v_cpu}
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        traffic = None
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_sweep")
            except Exception:
                traffic = None
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (device-generated, BASELINE config 2 shapes and distribution)" if device_generated
                     else f"synthetic (seeded CounterRng, BASELINE {args.config} shapes; random instance, no dataset)"),
            "config": config_block(arr, args.config, "yx monotone + FixedRestart(500) (rapdb-yx)",
                                   {"parallelism": (f"constraint-sharded over {ws} GPU(s), NCCL all-reduce per trial"
                                                    if sharded else ("replicas only" if ws > 1 else "single GPU")),
                                    "shard_range": None if shard is None else [shard.k0, shard.k1],
                                    "iterations_per_solve": results[-1].iterations,
                                    "evals_per_solve": results[-1].evals, "converged": conv,
                                    "final_kkt": results[-1].metrics.kkt_residual}),
            "time_to_kkt_ms": t_ms / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per sweep (dram__bytes_read.sum + dram__bytes_write.sum of one "
                                         "OP_PROBE sweep launch, ncu --set full, profiles/ncu_summary.json); "
                                         "achieved counts the same sweep bytes over the solve launch",
                         "traffic_over_algorithmic": (traffic / sweep_bytes) if traffic else None,
                         "peak_source": peak_src,
                         "kernel": "rapdb_solver_kernel (whole launch: sweeps + all other phases)",
                         "layout": layout,
                         "bytes_per_launch_def": ("sweeps x packed-symmetric stack bytes "
                                                  "(m+1) x rapdb_packed_doubles(n) x 8 (upper block triangle)"
                                                  if layout == "packed" else "sweeps x (m+1) n^2 8 B"),
                         "sweep_bytes": sweep_bytes,
                         "dense_equivalent_gbs": sweeps * dense_bytes / (kern_ms / 1e3) / 1e9,
                         "sweep_phase_gbs": sweep_phase_gbs,
                         "standalone_sweep_ms": probe_ms,
                         "standalone_sweep_gbs": None if probe_ms is None else sweep_bytes / (probe_ms / 1e3) / 1e9,
                         "frac_of_8tbs": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": e2e_block or {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                                 "d2h_bytes_per_step": int(d2h), "time_to_kkt_ms": 1e3 * e2e_s / args.steps},
            "nonmonotone": {"iters_per_s": rnm.iterations / tn, "iterations": rnm.iterations,
                            "evals": rnm.evals, "budget": 1000, "final_kkt": rnm.metrics.kkt_residual},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        emit(out)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
