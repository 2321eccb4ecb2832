"""APDB engine: drop-in for ``pkg/src/rapdb/engine.py`` backed by the device kernel.

``SolverConfig`` / ``TraceRecord`` / ``initial_iterate`` / ``run`` keep the
reference's signatures and semantics (engine.py:33-79, :275-294).
``ApdbEngine`` keeps its public surface (``step``, ``reinit``, ``last``,
``average``, ``trace``, ``iters``, ``evals_total``, ``T``, ``iterates``) but its
state lives in HBM: one ``step()`` is one launch of the persistent kernel
(``OP_RUN`` with ``max_iters=1``) that runs the whole backtracking loop on
device; ``run()`` issues all K iterations in a single launch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from . import _capi
from .errors import ConfigurationError
from .geometry import DualBall, Unbounded, project_set
from .problem import Iterate, ProblemInstance

GOLDEN_RATIO = 0.5 * (1.0 + math.sqrt(5.0))


@dataclass
class SolverConfig:
    mode: str = "yx"                      # "xy" or "yx"
    c_alpha: Optional[float] = None       # default 0.25 (xy) / 0.4 (yx)
    c_beta: Optional[float] = None        # default 0.3 (xy) / 0 (yx)
    delta: Optional[float] = None         # default 0.4 (xy) / 0.5 (yx)
    eta: float = 0.7
    tau_bar: float = 1.0
    gamma0: float = 1.0
    nonmonotone: bool = False
    dual_ball: DualBall = field(default_factory=Unbounded)
    max_backtracks: int = 200

    def resolved(self) -> "SolverConfig":
        """engine.py:46-63: mode defaults and validation."""
        if self.mode not in ("xy", "yx"):
            raise ConfigurationError(f"unknown mode {self.mode!r}")
        d = {"xy": (0.25, 0.3, 0.4), "yx": (0.4, 0.0, 0.5)}[self.mode]
        out = replace(self,
                      c_alpha=d[0] if self.c_alpha is None else self.c_alpha,
                      c_beta=d[1] if self.c_beta is None else self.c_beta,
                      delta=d[2] if self.delta is None else self.delta)
        if not (0.0 < out.eta < 1.0):
            raise ConfigurationError("eta must lie in (0, 1)")
        if out.tau_bar <= 0 or out.gamma0 <= 0:
            raise ConfigurationError("tau_bar and gamma0 must be positive")
        if out.c_alpha <= 0 or out.c_beta < 0 or not (0.0 < out.delta < 1.0):
            raise ConfigurationError("need c_alpha > 0, c_beta >= 0, delta in (0,1)")
        if out.mode == "xy" and out.c_beta <= 0:
            raise ConfigurationError("xy mode requires c_beta > 0")
        return out


@dataclass
class TraceRecord:
    iter: int
    tau_start: float
    tau: float
    sigma: float
    gamma: float
    evals_iter: int
    evals_total: int
    kkt: Optional[float] = None
    infeas: Optional[float] = None
    subopt: Optional[float] = None
    gap_xi: Optional[float] = None
    restart_flag: int = 0


def _opt(v):
    return None if v != v else float(v)  # NaN -> None


def records_from(rows: np.ndarray) -> List[TraceRecord]:
    out = []
    for r in rows:
        out.append(TraceRecord(iter=int(r[0]), tau_start=float(r[1]), tau=float(r[2]),
                               sigma=float(r[3]), gamma=float(r[4]), evals_iter=int(r[5]),
                               evals_total=int(r[6]), kkt=_opt(r[7]), infeas=_opt(r[8]),
                               subopt=_opt(r[9]), restart_flag=int(r[10])))
    return out


def _device_index(device):
    import torch
    if device is None:
        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    return torch.device(device).index or 0


class ApdbEngine:
    """One solver run whose state (iterates, U-cache, stepsize recursion,
    ergodic sums) is resident on the GPU."""

    def __init__(self, inst: ProblemInstance, config: SolverConfig, z_init: Iterate,
                 keep_iterates: bool = False, device=None, shard=None):
        """``shard`` (sharding.Shard): hold only matrices [k0, k1) and all-reduce
        the per-trial partials with the other ranks."""
        inst.check_device_support()
        self.inst = inst
        self.config = cfg = config.resolved()
        self.mu = inst.mu
        self.c_nm = 1.0 if cfg.nonmonotone else 0.0
        self.keep_iterates = keep_iterates
        self.trace: List[TraceRecord] = []
        self.iterates: List[Iterate] = []
        self.shard = shard
        idx = _device_index(device)
        if shard is None:
            self._ctx = _capi.Context(idx)
            self._data = inst.device_data(self._ctx.device)
            self._ctx.bind(self._data, cfg)
        else:
            self._ctx = _capi.Context(idx, shard.rank, shard.nranks)
            ctx = self._ctx
            if getattr(shard, "comm", None) is not None:     # native rank-ordered NCCL exchange
                ctx.set_comm_exchange(shard.comm, force_split=shard.split)
            else:
                ctx.set_exchange(lambda kind: shard.exchange(ctx.exchange_views(kind)), force_split=shard.split)
            if getattr(shard, "l0", None) is not None:
                self._data = inst.device_data(ctx.device, krange=(shard.k0, shard.k1), lrange=(shard.l0, shard.l1))
            else:
                self._data = inst.device_data(ctx.device, krange=(shard.k0, shard.k1))
            ctx.bind(self._data, cfg, shard.k0, shard.k1)
            if getattr(shard, "p2p", False) and not getattr(self._data, "factored", False):
                shard.attach_peer_exchange(ctx)
        self._trace_buf = None
        self._res = None
        self.iters = 0
        self.evals_total = 0
        self.reinit(z_init)

    # -- state management ------------------------------------------------
    def _tensor(self, a, size):
        torch = self._ctx.torch
        a = np.asarray(a, dtype=np.float64).reshape(-1)
        if a.shape != (size,):
            from .errors import InputError
            raise InputError(f"point of dim {a.shape} does not match {size}")
        if size == 0:
            return torch.zeros(1, dtype=torch.float64, device=self._ctx.device)
        return torch.from_numpy(a.copy()).to(self._ctx.device)

    def reinit(self, z: Iterate, warm_tau: bool = False):
        """engine.py:102-127 for an explicit host point."""
        x = self._tensor(z.x, self.inst.n)
        v = self._tensor(z.v, self.inst.p)
        lam = self._tensor(z.lam, self.inst.m)
        self._ctx.reinit(0, x, v, lam, warm_tau=warm_tau and self._res is not None, reset_inner=True)

    def reinit_from(self, source: str, warm_tau: bool = False):
        """Restart from the current iterate ("last") or the ergodic average,
        without a host round trip of the point."""
        self._ctx.reinit(1 if source == "last" else 2, warm_tau=warm_tau, reset_inner=True)

    def _buf(self, k):
        torch = self._ctx.torch
        if self._trace_buf is None or self._trace_buf.shape[0] < k:
            self._trace_buf = torch.empty((max(k, 64), _capi.TRACE_COLS), dtype=torch.float64,
                                          device=self._ctx.device)
        return self._trace_buf

    def _run(self, args: _capi.RunArgs):
        buf = self._buf(int(args.max_iters))
        try:
            res = self._ctx.run(args, buf)
        except Exception:
            raise
        self._res = res
        k = int(res.iters_done)
        rows = buf[:k].cpu().numpy() if k else np.zeros((0, _capi.TRACE_COLS))
        self.iters = int(res.total)
        self.evals_total = int(res.evals_total)
        return res, rows

    def run_block(self, k: int, **kw):
        """k accepted iterations in one launch (no KKT, no restarts)."""
        a = _capi.RunArgs(max_iters=k, budget=1 << 62, stop_total=0, metrics_every=0, criterion=0)
        for key, val in kw.items():
            setattr(a, key, val)
        res, rows = self._run(a)
        recs = records_from(rows)
        self.trace.extend(recs)
        return res, recs

    def run_block_args(self, args: _capi.RunArgs):
        res, rows = self._run(args)
        recs = records_from(rows)
        self.trace.extend(recs)
        return res, recs

    def smoothed_gap(self, source: int, xi: float, tol: float, x_warm=None, raw_point=None):
        """Device smoothed gap at the current iterate (1) or the ergodic average (2);
        returns (gap, Certificate, x_candidate_tensor)."""
        from .diagnostics import Certificate
        torch = self._ctx.torch
        x_cand = torch.empty(self.inst.n, dtype=torch.float64, device=self._ctx.device)
        point = None
        if raw_point is not None:
            source = 0
            point = (self._tensor(raw_point.x, self.inst.n), self._tensor(raw_point.v, self.inst.p),
                     self._tensor(raw_point.lam, self.inst.m))
        if x_warm is not None and not hasattr(x_warm, "data_ptr"):
            x_warm = self._tensor(x_warm, self.inst.n)
        out = self._ctx.smoothed_gap(source, xi, tol, x_warm, x_cand, point)
        self.last_gap = out
        return out[0], Certificate(int(out[1]), out[2], bool(out[3])), x_cand

    def step(self) -> TraceRecord:
        res, recs = self.run_block(1)
        if self.keep_iterates:
            self.iterates.append(self.last)
        return recs[-1]

    # -- scalar state (read back from the device after each launch) ------
    @property
    def T(self) -> float:
        return 0.0 if self._res is None else float(self._res.T)

    @property
    def tau_cand(self) -> float:
        return self.config.tau_bar if self._res is None else float(self._res.tau_cand)

    @property
    def gamma(self) -> float:
        return self.config.gamma0 if self._res is None else float(self._res.gamma)

    # -- results -----------------------------------------------------------
    def _fetch(self, which):
        x, v, lam = self._ctx.get_iterate(which)
        return Iterate(x.cpu().numpy(), v.cpu().numpy(), lam.cpu().numpy())

    @property
    def last(self) -> Iterate:
        return self._fetch(0)

    @property
    def z(self) -> Iterate:
        return self.last

    def average(self) -> Iterate:
        return self._fetch(1)


def initial_iterate(inst: ProblemInstance, dual_ball: DualBall = None) -> Iterate:
    """engine.py:275-283: projection of the origin (the device re-projects on reinit)."""
    x = project_set(inst.primal_set, np.zeros(inst.n))
    lam = inst.project_dual_cone(np.zeros(inst.m))
    v = np.zeros(inst.p)
    if dual_ball is not None:
        v, lam = dual_ball.project(v, lam)
    return Iterate(x, v, lam)


def run(inst: ProblemInstance, config: SolverConfig, z_init: Iterate, K: int,
        keep_iterates: bool = False):
    """K accepted iterations; returns (average, last, trace, engine) (engine.py:286-294)."""
    if K < 1:
        raise ConfigurationError("need K >= 1")
    engine = ApdbEngine(inst, config, z_init, keep_iterates=keep_iterates)
    if keep_iterates:
        for _ in range(K):
            engine.step()
    else:
        engine.run_block(K)
    return engine.average(), engine.last, engine.trace, engine


class _Evaluator:
    """Device evaluation of the operator contract at arbitrary points (used by
    coupling_value / grad_x_coupling / kkt_residual on user-given z)."""

    def __init__(self, inst: ProblemInstance):
        self.inst = inst
        self.ctx = _capi.Context(_device_index(None))
        self.data = inst.device_data(self.ctx.device)
        self.ctx.bind(self.data, SolverConfig().resolved())
        self._key = None
        self._val = None

    def _x(self, x):
        torch = self.ctx.torch
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(self.ctx.device)

    def sweep(self, x):
        x = np.asarray(x, dtype=np.float64)
        key = x.tobytes()
        if key != self._key:
            u, g, _ = self.ctx.probe_sweep(self._x(x))
            self._key, self._val = key, (u, g)
        return self._val

    def eq(self, x):
        """A x - b (problem.py:175-177) by the device probe sweep."""
        torch = self.ctx.torch
        out = torch.empty(max(self.inst.p, 1), dtype=torch.float64, device=self.ctx.device)
        self.ctx.eq_residual(self._x(x), out)
        return out[:self.inst.p]

    def kkt_at(self, z, f_star=None):
        """rapdb_kkt_at: the KKT metrics and Phi at z, all on the device."""
        inst = self.inst
        v = self._x(z.v) if inst.p else None
        lam = self._x(z.lam) if inst.m else None
        return self.ctx.kkt_at(self._x(z.x), v, lam, f_star)

    def coupling(self, z):
        """coupling_value (problem.py:196-204): (f + v.(Ax - b)) + lam.g."""
        return float(self.kkt_at(z)[8])

    def grad_x_t(self, z):
        """grad_x Phi(z) (problem.py:207-217) through the solver kernel's own
        recombination (rapdb_grad_x): dense U-cache or factored W-cache."""
        inst = self.inst
        v = self._x(z.v) if inst.p else None
        lam = self._x(z.lam) if inst.m else None
        gx, _ = self.ctx.grad_x(self._x(z.x), v, lam)
        return gx

    def grad_x(self, z):
        return self.grad_x_t(z).cpu().numpy()
