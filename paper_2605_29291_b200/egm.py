"""Extragradient baseline on the device (reference egm.py:1-92; SURVEY.md
section 8(f) row f4): a single constant stepsize for both blocks,

    z~ = Pi(z - s F(z)),  z+ = Pi(z - s F(z~)),  F = (grad_x Phi, -grad_y Phi),

Pi the product projection onto X times the (ball-capped) dual domain.  The
iterations run inside the persistent kernel (op EGM, csrc/egm.cuh) on the
same Q sweep, U-cache recombination and projections as rAPDB: two sweeps per
iteration, no host round trips.  Same signatures, result type, divergence
rule (|z| > 1e8 (1 + |z0|)), average and stepsize grid as the reference."""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _capi
from .engine import SolverConfig, _device_index
from .errors import ConfigurationError
from .geometry import DualBall, Unbounded
from .problem import Iterate

DEFAULT_STEP_GRID = tuple(np.logspace(-3, 0, 7))


@dataclass
class EgmResult:
    last: Iterate
    average: Iterate
    iterations: int
    diverged: bool
    trace: List[dict]


def run_egm(inst, stepsize: float, z_init: Iterate, K: int, dual_ball: DualBall = None,
            trace_every: int = 0, device=None) -> EgmResult:
    """egm.py:37-77 on the device."""
    if stepsize < 0:
        raise ConfigurationError("stepsize must be nonnegative")
    if K < 1:
        raise ConfigurationError("need K >= 1")
    if dual_ball is None:
        dual_ball = Unbounded()
    inst.check_device_support()
    ctx = _capi.Context(_device_index(device))
    data = inst.device_data(ctx.device)
    ctx.bind(data, SolverConfig(dual_ball=dual_ball).resolved())
    torch = ctx.torch

    def t(a, size):
        a = np.asarray(a, dtype=np.float64).reshape(-1)
        if size == 0:
            return torch.zeros(1, dtype=torch.float64, device=ctx.device)
        return torch.from_numpy(np.ascontiguousarray(a)).to(ctx.device)

    # the projection of z_init (egm.py:51) is the reinit's projection
    ctx.reinit(0, t(z_init.x, inst.n), t(z_init.v, inst.p), t(z_init.lam, inst.m))
    iters, diverged, tr = ctx.egm(float(stepsize), int(K), int(trace_every))

    def fetch(which):
        x, v, lam = ctx.get_iterate(which)
        return Iterate(x.cpu().numpy(), v.cpu().numpy(), lam.cpu().numpy())

    trace = [{"iter": int(r[0]), "norm": float(r[1])} for r in tr if 0 < int(r[0]) <= iters]
    res = EgmResult(last=fetch(0), average=fetch(1), iterations=iters, diverged=diverged, trace=trace)
    res._ctx = ctx      # the device context (diagnostics: guard checks)
    return res


def tune_egm(inst, z_init: Iterate, K: int, score, grid=DEFAULT_STEP_GRID,
             dual_ball: DualBall = None, device=None):
    """egm.py:80-92: the grid stepsize whose last iterate scores best (lower
    is better); returns (best_stepsize, best_result)."""
    best = None
    for s in grid:
        res = run_egm(inst, float(s), z_init, K, dual_ball=dual_ball, device=device)
        if res.diverged:
            continue
        val = score(res.last)
        if best is None or val < best[2]:
            best = (float(s), res, val)
    if best is None:
        raise ConfigurationError("every grid stepsize diverged")
    return best[0], best[1]
