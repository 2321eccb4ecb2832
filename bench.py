"""Benchmark: rAPDB on BASELINE.json config 1 (dense QCQP n=2000, m=200) on B200.

A "step" is one full drop-in solve, ``run_restarted`` of C1 to the conic
KKT / feasibility tolerance 1e-6 (``metrics_every=10``) with the reference
CLI's rapdb-yx policy (``FixedRestart(500)``, cli.py:90-107) and monotone
backtracking (the variant that converges on C1; the non-monotone variant is
timed on a fixed 1000-iteration budget and reported under ``nonmonotone``).

* ``value``        accepted iterations / s, Q stack resident in HBM.  N ranks
                   (torchrun, or ``--gpus N`` which launches torchrun itself):
                   the constraints are sharded over the GPUs and each trial
                   sums one n-vector and one (m+1)-vector across ranks with the
                   library's own rank-ordered NCCL exchange (csrc/comm.cuh;
                   ``scaling: strong``, one solve); ``--replicas`` runs
                   independent replicas instead (``scaling: weak``).
                   torch.distributed (gloo) is only the bootstrap / barrier.
* ``c2``           BASELINE C2 (n=4096, m=512, 69 GB dense / 34.7 GB packed),
                   generated on the device and sharded over the same N ranks:
                   it/s, time to KKT and sweep GB/s per GPU (the 6x target's basis).
* ``c3f``          BASELINE C3 (factored sparse, n = 10^6; feasible x0 variant) on
                   the same N ranks: it/s, time to KKT, time per test evaluation
                   against its HBM bytes and against the measured gather ceiling.
* ``ms_per_step``  = time-to-1e-6-KKT of one solve.
* ``e2e``          the same solve through the public API with the instance on
                   the HOST: pinned H2D of the 6.4 GB Q stack + vectors, solve,
                   D2H of solution/average/trace/metrics, all inside the timing.
* ``roofline``     the solver kernel: algorithmic Q bytes streamed (sweeps x
                   (m+1) n^2 8 B) / CUDA-event duration of its launches.
* ``cpu_baseline`` the CPU oracle (numpy restatement of the reference, same
                   arithmetic and matvec count) solving the same C1 arrays TO KKT
                   with the same policy (wall-capped), on the host's cores.

``--impl reference`` times that CPU restatement alone, to KKT, the timed
iterations split into K steps (the reference is pure Python: nothing is
compiled into oracle/_ref).  Inputs (6.4 GB) exceed the
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
    ap.add_argument("--cpu-cap-s", type=float, default=240.0,
                    help="wall-clock cap of the CPU solve to KKT (reported as not converged beyond it)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--c2-steps", type=int, default=1, help="timed C2 solves (0: no c2 block)")
    ap.add_argument("--c3-steps", type=int, default=1, help="timed C3f solves (0: no c3f block)")
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


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"cpu_model": model, "affinity_cores": aff, "blas_threads": blas_threads(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


class _Cap(Exception):
    pass


def oracle_to_kkt(arr, cap_s, marks=None):
    """The CPU port (oracle/rapdb_oracle.py, the reference's arithmetic and
    matvec count) solving `arr` to conic KKT 1e-6 with the bench policy
    (yx monotone + FixedRestart(500), KKT every 10 iterations), stopped at
    `cap_s` seconds of wall time.  marks: list receiving (iteration, t)."""
    from oracle import rapdb_oracle as O
    P = O.Problem.from_arrays(arr)
    t0 = time.perf_counter()
    state = {"it": 0}

    def hook(total, eng):
        state["it"] = total
        now = time.perf_counter() - t0
        if marks is not None:
            marks.append((total, now))
        if now > cap_s:
            raise _Cap()

    converged = False
    try:
        res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=False), O.Policy(kind="fixed", period=500),
                              budget=50_000, criteria=dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6),
                              metrics_every=10, on_iter=hook)
        converged = bool(res.converged)
        iters = res.iterations
    except _Cap:
        iters = state["it"]
    dt = time.perf_counter() - t0
    return iters, dt, converged


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
    marks = []
    iters, dt, conv = oracle_to_kkt(arr, args.cpu_cap_s, marks)
    # warm-up = the first W accepted iterations (includes the initial
    # backtracking from tau_bar); the rest of the solve is split into K steps
    w = min(max(args.warmup, 0), max(iters - 1, 0))
    t_w = marks[w - 1][1] if w > 0 else 0.0
    timed_iters = iters - w
    timed_s = dt - t_w
    v = timed_iters / timed_s if timed_s > 0 else None
    info = host_info()
    sample = (f"port (oracle/rapdb_oracle.py) solving {args.config} to conic KKT 1e-6, yx monotone + "
              f"FixedRestart(500): {iters} iterations in {dt:.1f} s ({'converged' if conv else 'wall cap hit'}); "
              f"the first {w} iterations are the warm-up, the remaining {timed_iters} are timed as "
              f"{args.steps} steps")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * timed_s / max(args.steps, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded CounterRng, BASELINE config shapes)",
           "config": config_block(arr, args.config, "yx monotone + FixedRestart(500) (rapdb-yx), to KKT"),
           "time_to_kkt_s": dt if conv else None, "converged": conv, "iterations": iters,
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": info["blas_threads"], "kind": "port",
                            "sample": sample, **info},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`--gpus N` outside torchrun: launch N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_dist(ws, local, need_group):
    """torch.distributed (gloo) as plumbing only: the NCCL unique-id bootstrap,
    barriers and the max-over-ranks of the timings.  The data path's
    exchanges run in the library over its own NCCL communicator."""
    import torch
    torch.cuda.set_device(local)
    if not need_group:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("gloo")
    return dist


class Ranks:
    def __init__(self, dist, dev):
        self.dist, self.dev = dist, dev

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()

    def reduce(self, v, op):
        if self.dist is None:
            return v
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        self.dist.all_reduce(t, op=op(self.dist))
        return float(t.item())

    def max(self, v):
        return self.reduce(v, lambda d: d.ReduceOp.MAX)

    def min(self, v):
        return self.reduce(v, lambda d: d.ReduceOp.MIN)

    def sum(self, v):
        return self.reduce(v, lambda d: d.ReduceOp.SUM)


def timed_solves(R, inst, cfg, pol, crit, dev, shard, ranks, steps, warmup, budget=50_000):
    """W untimed + K timed solves, CUDA events on the launching stream, max over ranks."""
    import torch

    def solve():
        return R.run_restarted(inst, cfg, pol, budget=budget, criteria=crit, metrics_every=10, device=dev,
                               shard=shard)
    for _ in range(warmup):
        solve()
    ranks.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    results = [solve() for _ in range(steps)]
    ev1.record()
    ranks.barrier()
    return results, ranks.max(ev0.elapsed_time(ev1))


def sweep_stats(results):
    kern_ms = sum(r.device_stats["kernel_ms"] for r in results)
    sweeps = sum(r.device_stats["sweeps"] for r in results)
    sweep_ns = sum(r.device_stats["sweep_ns"] for r in results)
    sweep_bytes = results[-1].device_stats["sweep_bytes"]
    return kern_ms, sweeps, sweep_ns, sweep_bytes


def c2_block(R, args, dev, shard_fn, ranks, ws, peak):
    """BASELINE C2 sharded over the job's ranks (device-generated stack)."""
    import torch
    inst = R.DeviceDenseInstance(4096, 512, 256, seed=0, name="C2 (device-generated)")
    shard = shard_fn(inst)
    krange = None if shard is None else (shard.k0, shard.k1)
    t0 = time.perf_counter()
    inst.device_data(dev, krange=krange)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    cfg = R.SolverConfig(mode="yx", nonmonotone=False)
    crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    results, t_ms = timed_solves(R, inst, cfg, R.FixedRestart(500), crit, dev, shard, ranks,
                                 args.c2_steps, 1)
    kern_ms, sweeps, sweep_ns, sweep_bytes = sweep_stats(results)
    local_gbs = sweeps * sweep_bytes / (kern_ms / 1e3) / 1e9
    local_sweep_gbs = sweeps * sweep_bytes / sweep_ns
    its = results[-1].iterations
    out = {"workload": "C2: dense convex QCQP n=4096, m=512, B_i rank 256 (device-generated, same "
                       "distribution as BASELINE config 2), 68.85 GB dense / 34.70 GB packed fp64",
           "policy": "yx monotone + FixedRestart(500), conic KKT 1e-6",
           "n_gpus": ws, "shard_range": None if shard is None else [shard.k0, shard.k1],
           "iters_per_s": its * args.c2_steps / (t_ms / 1e3), "time_to_kkt_ms": t_ms / args.c2_steps,
           "iterations": its, "evals": results[-1].evals, "converged": bool(results[-1].converged),
           "final_kkt": results[-1].metrics.kkt_residual,
           "sweep_bytes_per_gpu_max": ranks.max(sweep_bytes),
           "kernel_gbs_per_gpu_min": ranks.min(local_gbs),
           "sweep_phase_gbs_per_gpu_min": ranks.min(local_sweep_gbs),
           "roofline_frac_min": ranks.min(local_gbs) / peak,
           "sweep_phase_frac_min": ranks.min(local_sweep_gbs) / peak,
           "generate_s": gen_s, "steps": args.c2_steps, "warmup": 1}
    inst.drop_device_data()
    return out


def c3f_block(R, args, dev, shard_fn, ranks, ws, peak):
    """BASELINE C3 (factored sparse, n = 10^6) with x0 ~ U(-0.01, 0.01) -- the
    config's own x0 ~ U(-1, 1) admits no feasible point (tools/c3_infeasibility.py)
    -- constraint-sharded over the job's ranks.  Per test evaluation the path
    gathers 2 (nnz R + nnz A) doubles (one L1 line lookup each: the bound of
    the sparse passes, tools/gather_probe.cu) and streams eval_bytes from HBM."""
    import torch
    from paper_2605_29291_b200 import instances
    t0 = time.perf_counter()
    arr = instances.factored_qcqp(x0_scale=0.01)
    inst = R.FactoredInstance.from_arrays(arr)
    shard = shard_fn(inst)
    kw = {} if shard is None else {"krange": (shard.k0, shard.k1), "lrange": (shard.l0, shard.l1)}
    inst.device_data(dev, **kw)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    cfg = R.SolverConfig(mode="yx", nonmonotone=False)
    crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    results, t_ms = timed_solves(R, inst, cfg, R.FixedRestart(500), crit, dev, shard, ranks,
                                 args.c3_steps, 1, budget=5000)
    res = results[-1]
    nnz_r, nnz_a = int(inst.R.nnz), int(inst.A.nnz)
    eval_bytes = 2 * 12 * nnz_r + 2 * 8 * (inst.mq + 1) * inst.n + 2 * 12 * nnz_a
    gathers = 2 * (nnz_r + nnz_a)
    evals = sum(r.evals for r in results)
    per_eval_s = (t_ms / 1e3) / max(evals, 1)
    ceiling = None
    probe = os.path.join(ROOT, "profiles", "r02c_gather_probe.json")
    if os.path.exists(probe):
        try:
            rows = json.load(open(probe))["results"]
            ceiling = max(r["ggather_s"] for r in rows if r["variant"].startswith("ldg8idx"))
        except Exception:
            ceiling = None
    out = {"workload": "C3f: factored sparse QCQP n=1e6, 64 quadratic rows R_i^T R_i (1e5 x n, 10 nnz/row), "
                       "5e5 linear rows (5 nnz), x0 ~ U(-0.01, 0.01)",
           "policy": "yx monotone + FixedRestart(500), conic KKT 1e-6",
           "n_gpus": ws, "shard_range": None if shard is None else [shard.k0, shard.k1, shard.l0, shard.l1],
           "iters_per_s": res.iterations * args.c3_steps / (t_ms / 1e3), "time_to_kkt_ms": t_ms / args.c3_steps,
           "iterations": res.iterations, "evals": res.evals, "converged": bool(res.converged),
           "final_kkt": res.metrics.kkt_residual, "us_per_eval": 1e6 * per_eval_s,
           "eval_bytes": eval_bytes, "eval_gbs": eval_bytes / ws / per_eval_s / 1e9,
           "eval_frac_of_hbm_peak": eval_bytes / ws / per_eval_s / 1e9 / peak,
           "gathers_per_eval": gathers, "ggather_s": gathers / ws / per_eval_s / 1e9,
           "gather_ceiling_ggather_s": ceiling,
           "frac_of_gather_ceiling": None if not ceiling else gathers / ws / per_eval_s / 1e9 / ceiling,
           "bound": "L1 wavefront rate of the 8-byte gathers (whole trial incl. control steps and launch gaps "
                    "over the gathers alone); HBM bytes are below the stream's time",
           "generate_upload_s": gen_s, "steps": args.c3_steps, "warmup": 1}
    inst.drop_device_data()
    return out


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    _claim_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    if torch.cuda.device_count() < max(ws, 1) and ws > 1:
        raise SystemExit(f"{ws} ranks need {ws} GPUs, {torch.cuda.device_count()} visible")
    sharded = (ws > 1 and not args.replicas) or args.shard
    os.environ.setdefault("NCCL_DEBUG", "INFO")        # communicator lines go to stderr (_claim_stdout)
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist = init_dist(ws, local, ws > 1 or args.shard)
    dev = torch.device("cuda", torch.cuda.current_device())
    ranks = Ranks(dist, dev)

    import paper_2605_29291_b200 as R
    from paper_2605_29291_b200 import _capi, instances
    from paper_2605_29291_b200.sharding import nccl_shard

    def shard_fn(inst):
        if not sharded:
            return None
        sh = nccl_shard(inst, device_index=dev.index)
        sh.force_split = True
        sh.p2p = bool(args.p2p)
        return sh

    device_generated = args.config == "C2"
    if device_generated:
        inst = R.DeviceDenseInstance(4096, 512, 256, seed=0, name="C2 (device-generated)")
        arr = inst
    else:
        arr = instances.config_instance(args.config)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
    cfg = R.SolverConfig(mode="yx", nonmonotone=False)
    pol = R.FixedRestart(500)
    crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    shard = shard_fn(inst)
    krange = None if shard is None else (shard.k0, shard.k1)
    inst.device_data(dev, krange=krange)
    peak, peak_src = measured_peak()

    # ---- device-resident timed region -----------------------------------
    clocks = ClockSampler(torch.cuda.current_device())
    launches0 = _capi.launch_count()
    clocks.start()
    results, t_ms = timed_solves(R, inst, cfg, pol, crit, dev, shard, ranks, args.steps, args.warmup)
    clk = clocks.stop()
    launches = _capi.launch_count() - launches0
    iters_local = sum(r.iterations for r in results)
    # sharded: every rank runs the same solve (strong scaling); replicas: sum
    iters_all = iters_local if sharded else ranks.sum(iters_local)
    value = iters_all / (t_ms / 1e3)
    conv = all(r.converged for r in results)
    kern_ms, sweeps, sweep_ns, sweep_bytes = sweep_stats(results)
    layout = os.environ.get("RAPDB_LAYOUT", "packed")
    dense_bytes = (arr.m + 1 if shard is None else shard.k1 - shard.k0) * arr.n * arr.n * 8
    achieved = sweeps * sweep_bytes / (kern_ms / 1e3) / 1e9
    sweep_phase_gbs = sweeps * sweep_bytes / sweep_ns

    # standalone sweep launch (one kernel launch = one fused sweep), CUDA events
    probe_ms = None
    if shard is None:
        ev = inst._evaluator()
        xprobe = torch.from_numpy(np.asarray(results[-1].solution.x)).to(dev)
        ev.ctx.probe_sweep(xprobe, reps=1)
        _, _, probe_ms = ev.ctx.probe_sweep(xprobe, reps=10)

    # ---- e2e through the public API with host-resident inputs -----------
    e2e_block = None
    if device_generated:
        e2e_block = {"unavailable": "device-generated instance: its inputs never exist on the host"}
    else:
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
        ranks.barrier()
        t0 = time.perf_counter()
        r = R.run_restarted(inst, cfg, pol, budget=50_000, criteria=crit, metrics_every=10, device=dev,
                            shard=shard)
        sol = (r.solution.x, r.average.x)     # noqa: F841 -- the D2H reads are part of the call
        ranks.barrier()
        e2e_s += time.perf_counter() - t0
        e2e_iters += r.iterations
        # solution + average (x, v, lam), the trace rows and the metrics
        d2h = 2 * (arr.n + arr.m + arr.p) * 8 + r.iterations * 11 * 8 + 8 * 8
    e2e_s = ranks.max(e2e_s)
    e2e_value = (e2e_iters if sharded else ranks.sum(e2e_iters)) / e2e_s if e2e_s > 0 else None

    # non-monotone variant: fixed 1000-iteration budget (it/s only)
    inst.device_data(dev, krange=krange)
    nm_cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    ranks.barrier()
    tn = time.perf_counter()
    rnm = R.run_restarted(inst, nm_cfg, pol, budget=1000, criteria=crit, metrics_every=10, device=dev,
                          shard=shard)
    ranks.barrier()
    tn = ranks.max(time.perf_counter() - tn)
    if not device_generated:
        inst.drop_device_data()

    # the side blocks must not take the headline line down with them (single
    # rank only: in a sharded job a rank that skipped a block would leave the
    # others waiting in its collectives, so there a failure stays fatal)
    def guarded(fn):
        if ws > 1:
            return fn(R, args, dev, shard_fn, ranks, ws, peak)
        try:
            return fn(R, args, dev, shard_fn, ranks, ws, peak)
        except Exception as exc:   # noqa: BLE001
            import traceback
            traceback.print_exc()
            torch.cuda.empty_cache()
            return {"error": f"{type(exc).__name__}: {exc}"[:300]}

    c2 = None
    if args.c2_steps > 0 and not device_generated:
        c2 = guarded(c2_block)

    c3f = None
    if args.c3_steps > 0 and not device_generated:
        c3f = guarded(c3f_block)

    if rank == 0:
        cpu = None
        if not args.skip_cpu and ws == 1 and not device_generated:
            iters_c, dt_c, conv_c = oracle_to_kkt(arr, args.cpu_cap_s)
            info = host_info()
            cpu = {"value": iters_c / dt_c, "unit": UNIT, "cores": info["blas_threads"], "kind": "port",
                   "sample": (f"port (oracle/rapdb_oracle.py: the reference's arithmetic and matvec count) "
                              f"solving the same {args.config} arrays to conic KKT 1e-6 with the same policy: "
                              f"{iters_c} iterations in {dt_c:.1f} s"
                              + ("" if conv_c else f" (wall cap {args.cpu_cap_s:.0f} s hit, not converged)")),
                   "time_to_kkt_s": dt_c if conv_c else None, "converged": conv_c, "iterations": iters_c,
                   **info}
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
                                   {"parallelism": (f"constraint-sharded over {ws} GPU(s), rank-ordered NCCL "
                                                    f"exchange per trial (library-owned communicator)"
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
            "c2": c2,
            "c3f": c3f,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        emit(out)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
