"""Restart envelopes: drop-in for ``pkg/src/rapdb/restarts.py``.

``run_restarted`` keeps the reference signature and ordering
(restarts.py:82-170): step -> inner += 1 -> KKT + termination every
``metrics_every`` (or at ``total == budget``) -> fixed / adaptive restart.
The device executes the loop body; the host only wakes up when the kernel
returns: convergence, budget, an adaptive-restart gap check (the host decides
the restart from the device-computed gap), or a fixed restart whose point the
caller asked to record.
"""

from __future__ import annotations

import os

from dataclasses import dataclass
from typing import List, Optional, Union

from . import _capi, diagnostics
from .engine import ApdbEngine, SolverConfig, TraceRecord, initial_iterate
from .errors import ConfigurationError
from .problem import Iterate, ProblemInstance


@dataclass(frozen=True)
class NoRestart:
    pass


@dataclass(frozen=True)
class FixedRestart:
    period: int
    point: str = "last"

    def __post_init__(self):
        if self.period < 1:
            raise ConfigurationError("restart period must be >= 1")
        if self.point not in ("last", "average"):
            raise ConfigurationError("restart point must be 'last' or 'average'")


@dataclass(frozen=True)
class AdaptiveRestart:
    xi: float = 0.04
    q: float = 0.5
    warmup: int = 50
    check_period: int = 200
    point: str = "last"

    def __post_init__(self):
        if self.xi <= 0 or not (0.0 < self.q < 1.0):
            raise ConfigurationError("need xi > 0 and q in (0, 1)")
        if self.warmup < 1 or self.check_period < 1:
            raise ConfigurationError("warmup and check_period must be >= 1")
        if self.point not in ("last", "average"):
            raise ConfigurationError("restart point must be 'last' or 'average'")


RestartPolicy = Union[NoRestart, FixedRestart, AdaptiveRestart]


@dataclass
class RestartEvent:
    outer: int
    iteration: int
    trigger: str
    gap_new: Optional[float] = None
    gap_ref: Optional[float] = None
    point: Optional[Iterate] = None


@dataclass
class RunResult:
    solution: Iterate
    average: Iterate
    trace: List[TraceRecord]
    restart_log: List[RestartEvent]
    iterations: int
    evals: int
    converged: bool
    status: str
    metrics: Optional[diagnostics.Metrics] = None
    device_stats: Optional[dict] = None


def _next_check(policy: AdaptiveRestart, total: int, inner: int, gap_ref) -> int:
    """First total > `total` at which restarts.py:137-141 fires."""
    if gap_ref is None:
        return max(policy.warmup, total + 1)
    cp = policy.check_period
    nxt_inner = (inner // cp + 1) * cp
    return total + (nxt_inner - inner)


def run_restarted(inst: ProblemInstance, config: SolverConfig,
                  policy: RestartPolicy = None, z_init: Optional[Iterate] = None,
                  budget: int = 50_000,
                  criteria: Optional[diagnostics.TerminationCriteria] = None,
                  metrics_every: int = 10, warm_tau: bool = False,
                  record_restart_points: bool = False, device=None, shard=None) -> RunResult:
    """restarts.py:82-170.  Extra keyword arguments (not in the reference):
    ``device`` picks the GPU; ``shard`` (sharding.Shard, e.g. from
    ``sharding.nccl_shard(inst)`` in a torchrun job) shards the constraints over
    ranks -- every rank calls run_restarted with the same arguments."""
    if budget < 1:
        raise ConfigurationError("budget must be >= 1")
    if policy is None:
        policy = NoRestart()
    config = config.resolved()
    crit_code = 0 if criteria is None else criteria.code()
    if z_init is None:
        z_init = initial_iterate(inst, config.dual_ball)
    engine = ApdbEngine(inst, config, z_init, device=device, shard=shard)
    restart_log: List[RestartEvent] = []
    outer = 0
    inner = 0
    gap_ref = None
    x_warm = None
    converged = False
    status = "budget"
    metrics = None
    total = 0
    stats = {"sweep_ns": 0.0, "sweeps": 0, "kernel_ms": 0.0, "run_launches": 0, "sweep_bytes": 0}

    while total < budget:
        a = _capi.RunArgs(max_iters=budget - total, budget=budget, stop_total=0,
                          metrics_every=metrics_every if criteria is not None else 0,
                          criterion=crit_code)
        if criteria is not None:
            a.eps = criteria.eps
            a.eps_kkt = criteria.eps_kkt
            a.eps_feas = criteria.eps_feas
            if criteria.f_star is not None:
                a.f_star = criteria.f_star
                a.has_f_star = 1
        if isinstance(policy, FixedRestart):
            a.fixed_period = policy.period
            a.fixed_point = 1 if policy.point == "average" else 0
            a.warm_tau = 1 if warm_tau else 0
            a.stop_at_fixed = 1 if record_restart_points else 0
        elif isinstance(policy, AdaptiveRestart):
            nxt = _next_check(policy, total, inner, gap_ref)
            a.stop_total = nxt if nxt < budget else 0
        res, recs = engine.run_block_args(a)
        stats["sweep_ns"] += res.sweep_ns
        stats["sweeps"] += int(res.sweeps)
        stats["kernel_ms"] += res.kernel_ms
        stats["run_launches"] += 1
        stats["sweep_bytes"] = int(res.sweep_bytes)
        for r in recs:                      # fixed restarts executed on device
            if r.restart_flag:
                outer += 1
                restart_log.append(RestartEvent(outer=outer, iteration=r.iter, trigger="fixed"))
        total = int(res.total)
        inner = int(res.inner)
        if res.has_metrics and criteria is not None:
            metrics = diagnostics.metrics_from(list(res.metrics), criteria.f_star)
        if res.status == _capi.RUN_CONVERGED:
            converged, status = True, "converged"
            break
        if res.status in (_capi.RUN_BUDGET, _capi.RUN_LIMIT):
            break
        rec = engine.trace[-1]
        if res.status == _capi.RUN_FIXED_DUE:
            z_r = engine.last if policy.point == "last" else engine.average()
            engine.reinit_from(policy.point, warm_tau=warm_tau)
            outer += 1
            rec.restart_flag = 1
            restart_log.append(RestartEvent(outer=outer, iteration=total, trigger="fixed",
                                            point=z_r if record_restart_points else None))
            inner = 0
        elif res.status == _capi.RUN_CHECK_DUE:
            tol = 1e-9 if gap_ref is None else min(
                1e-9, 0.01 * policy.xi * max(gap_ref, 0.0) + 1e-15)
            gap_new, cert, x_cand = engine.smoothed_gap(
                1 if policy.point == "last" else 2, policy.xi, tol, x_warm)
            x_warm = x_cand
            rec.gap_xi = gap_new
            if gap_ref is None:
                gap_ref = gap_new
            elif gap_new <= policy.q * gap_ref:
                z_c = (engine.last if policy.point == "last" else engine.average()) \
                    if record_restart_points else None
                engine.reinit_from(policy.point, warm_tau=warm_tau)
                outer += 1
                inner = 0
                rec.restart_flag = 1
                restart_log.append(RestartEvent(outer=outer, iteration=total, trigger="adaptive",
                                                gap_new=gap_new, gap_ref=gap_ref, point=z_c))
                gap_ref = gap_new

    if metrics is None:
        f_star = criteria.f_star if criteria is not None else None
        metrics = diagnostics.metrics_from(engine._ctx.kkt(f_star), f_star)
    if os.environ.get("RAPDB_STEP_PROFILE", "0") == "1":
        stats["step_profile"] = engine._ctx.step_profile()
    return RunResult(solution=engine.last, average=engine.average(), trace=engine.trace,
                     restart_log=restart_log, iterations=engine.iters, evals=engine.evals_total,
                     converged=converged, status=status, metrics=metrics,
                     device_stats=stats)
