"""Solution-quality metrics: drop-in for ``pkg/src/rapdb/diagnostics.py``.

Inside ``run_restarted`` the KKT residual (diagnostics.py:96-113) and the
termination test (:252-263) run in the persistent kernel every
``metrics_every`` iterations, from the cached U = [Q_i x_k] (no extra sweep).
The standalone functions below evaluate at a user-given point on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigurationError
from .problem import Iterate, ProblemInstance


@dataclass
class Metrics:
    kkt_residual: float
    stationarity: float
    primal_eq: float
    complementarity: float
    infeas: float
    f_value: float
    mean_pos_violation: float
    subopt_abs: Optional[float] = None
    gap_xi: Optional[float] = None
    gap_reliable: bool = True


@dataclass
class TerminationCriteria:
    eps: float = 1e-7
    f_star: Optional[float] = None
    criterion: str = "paper51"
    eps_kkt: float = 1e-7
    eps_feas: float = 1e-7

    def code(self) -> int:
        if self.criterion == "conic":
            return 1
        if self.criterion == "paper51":
            return 2
        raise ConfigurationError(f"unknown termination criterion {self.criterion!r}")


@dataclass
class Certificate:
    iterations: int
    residual: float
    converged: bool


def metrics_from(vals, f_star=None) -> Metrics:
    return Metrics(kkt_residual=vals[0], stationarity=vals[1], primal_eq=vals[2],
                   complementarity=vals[3], infeas=vals[4], f_value=vals[5],
                   mean_pos_violation=vals[6],
                   subopt_abs=None if f_star is None else vals[7])


def kkt_residual(inst: ProblemInstance, z: Iterate, f_star: Optional[float] = None) -> Metrics:
    """r(x, v, lam) at an arbitrary point (diagnostics.py:96-113), evaluated on
    the device in one op (rapdb_kkt_at: sweep, g, grad_x Phi, the norms)."""
    vals = inst._evaluator().kkt_at(z, f_star)
    return metrics_from(vals, f_star)


def infeasibility(inst: ProblemInstance, x) -> float:
    return kkt_residual(inst, Iterate(x, np.zeros(inst.p), np.zeros(inst.m))).infeas


def mean_positive_violation(inst: ProblemInstance, x) -> float:
    """diagnostics.py:57-66 for the orthant cone: (1/m) sum_i max(g_i(x), 0),
    with g evaluated by a device sweep."""
    if inst.m == 0:
        return 0.0
    g = np.asarray(inst.g_value(x), dtype=float)
    return float(np.mean(np.maximum(g, 0.0)))


def check_termination(metrics: Metrics, criteria: TerminationCriteria) -> bool:
    """diagnostics.py:252-263 (the same predicate the kernel evaluates)."""
    if criteria.criterion == "paper51":
        if criteria.f_star is None:
            return (metrics.kkt_residual <= criteria.eps_kkt
                    and metrics.infeas <= criteria.eps_feas)
        rel_gap = abs(metrics.f_value - criteria.f_star) / (1.0 + abs(criteria.f_star))
        return max(rel_gap, metrics.mean_pos_violation) <= criteria.eps
    if criteria.criterion == "conic":
        return (metrics.kkt_residual <= criteria.eps_kkt
                and metrics.infeas <= criteria.eps_feas)
    raise ConfigurationError(f"unknown termination criterion {criteria.criterion!r}")


def smoothed_gap(inst: ProblemInstance, z: Iterate, xi: float, dual_ball=None,
                 subsolver_tol: float = 1e-9, x_warm=None):
    """G_xi(z) (diagnostics.py:120-163) on the device; returns (gap, Certificate)."""
    from .engine import ApdbEngine, SolverConfig
    from .geometry import Unbounded
    if xi <= 0:
        raise ConfigurationError("xi must be positive")
    ball = dual_ball or Unbounded()
    # one bound gap engine per (instance, dual ball), reused across calls like
    # inst._evaluator(): the point is passed raw, the engine's own iterate is unused
    cache = getattr(inst, "_dev", None)
    key = ("_gap", repr(ball))
    eng = cache.get(key) if cache is not None else None
    if eng is None:
        eng = ApdbEngine(inst, SolverConfig(dual_ball=ball), z)
        if cache is not None:
            cache[key] = eng
    gap, cert, _ = eng.smoothed_gap(1, xi, subsolver_tol, x_warm, raw_point=z)
    return gap, cert
