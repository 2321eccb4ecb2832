"""CPU oracle: numpy restatement of the reference rAPDB hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker (or as the timed CPU baseline).  The product
package never imports it and has no CPU fallback.

What it restates (all citations are ``pkg/src/rapdb/<file>:<line>`` of the
reference at /root/reference):

* operator contract -- ``problem.py:166-180`` (f, g, Ax-b), ``problem.py:196-223``
  (Phi, grad_x Phi, grad_y Phi) and the dense/CSR storage rule ``problem.py:28-40``;
* ``ApdbEngine`` -- ``engine.py:86-272``: reinit/caches, both test functions,
  both candidate steps, the backtracking ``step`` and the ergodic average;
* ``run_restarted`` -- ``restarts.py:82-170`` with No/Fixed/Adaptive policies;
* diagnostics -- ``diagnostics.py:49-113`` (KKT, infeasibility, complementarity
  for the orthant), ``diagnostics.py:120-163`` (smoothed gap),
  ``diagnostics.py:252-263`` (termination);
* ``subsolve.py:27-62`` (APG with function-value restart) and
  ``problem.py:47-68`` (power-iteration spectral norm).

Every floating-point expression keeps the reference's operation order and its
numpy calls (``Q @ x`` dgemv, ``x @ y`` ddot, ``np.linalg.norm``), so on one
machine the oracle reproduces the reference bit for bit; that is what
``tests/test_oracle_pin.py`` checks against the committed golden traces made by
``tests/golden/make_golden.py`` from the real reference.

Deliberately literal: it recomputes Q-stack products the way the reference
does (about five stack sweeps per yx trial), so its timing is the reference
CPU cost that ``bench.py`` reports as the baseline.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.sparse as sp

GOLDEN_RATIO = 0.5 * (1.0 + np.sqrt(5.0))


class OracleError(RuntimeError):
    pass


class OracleNonConvergence(OracleError):
    def __init__(self, msg, state):
        super().__init__(msg)
        self.state = state


def _storage(M, n):
    """problem.py:31-40: CSR when fewer than 25% of the entries are nonzero."""
    if sp.issparse(M) or not isinstance(M, np.ndarray):
        return M
    M = np.asarray(M, dtype=float)
    if n > 0 and np.count_nonzero(M) < 0.25 * M.size:
        return sp.csr_matrix(M)
    return M


class FactoredOp:
    """Q = R^T R applied as R^T (R x): the config-3 restatement of a factored
    quadratic form.  Held by ``Problem`` like any
    other operator (problem.py:31-40 keeps non-array operators as given)."""

    def __init__(self, R):
        self.R = sp.csr_matrix(R)
        self.RT = self.R.T.tocsr()
        self.shape = (self.R.shape[1], self.R.shape[1])

    def __matmul__(self, x):
        return self.RT @ (self.R @ x)


class FactoredProblem:
    """Large-size config-3 restatement: quadratic rows as FactoredOp, the
    linear block vectorised (g = A x - b, grad += A^T mu) instead of L explicit
    dense q rows.  Same mathematics as ``factored_problem``; summation order of
    the linear rows differs, so it is compared to the device within tolerance."""

    def __init__(self, arr):
        self.n, self.mq, self.L = arr.n, arr.mq, arr.L
        self.m = arr.mq + arr.L
        self.p = 0
        self.Qf = [FactoredOp(arr.block(i)) for i in range(arr.mq + 1)]
        self.C = [np.asarray(arr.C[i]) for i in range(arr.mq + 1)]
        self.d = np.asarray(arr.d, dtype=float)
        self.A = sp.csr_matrix(arr.A)
        self.AT = self.A.T.tocsr()
        self.bl = np.asarray(arr.b, dtype=float)
        self.lo = np.asarray(arr.lower, dtype=float)
        self.hi = np.asarray(arr.upper, dtype=float)
        self.mu = 0.0
        self.b = np.zeros(0)

    def f(self, x):
        return 0.5 * float(x @ (self.Qf[0] @ x)) + float(self.C[0] @ x) + self.d[0]

    def g(self, x):
        quad = [0.5 * float(x @ (self.Qf[i] @ x)) + float(self.C[i] @ x) + self.d[i]
                for i in range(1, self.mq + 1)]
        return np.concatenate([np.array(quad), self.A @ x - self.bl])

    def eq(self, x):
        return np.zeros(0)

    def clip(self, w):
        return np.clip(w, self.lo, self.hi)

    def phi(self, x, v, lam):
        return self.f(x) + (float(lam @ self.g(x)) if self.m > 0 else 0.0)

    def grad_x(self, x, v, lam):
        out = self.Qf[0] @ x + self.C[0]
        for i in range(self.mq):
            w = lam[i]
            if w != 0.0:
                out = out + w * (self.Qf[i + 1] @ x + self.C[i + 1])
        if self.L:
            out = out + self.AT @ lam[self.mq:]
        return out


def factored_problem(arr, dense=False):
    """Oracle Problem for an ``instances.FactoredArrays``: Q_i = R_i^T R_i as
    FactoredOp (or, ``dense=True``, the explicit products exactly as the
    reference is given them, see FactoredArrays.dense_lists), Q = 0 (empty
    CSR, problem.py:38-39) for the linear rows, q = (C, rows of A), r = (d, -b)."""
    if dense:
        Q, q, r = arr.dense_lists()
    else:
        Q = [FactoredOp(arr.block(i)) for i in range(arr.mq + 1)]
        Q += [sp.csr_matrix((arr.n, arr.n)) for _ in range(arr.L)]
        Ad = arr.A.toarray()
        q = [arr.C[i] for i in range(arr.mq + 1)] + [Ad[j] for j in range(arr.L)]
        r = np.concatenate([arr.d, -arr.b])
    return Problem(Q, q, r, np.zeros((0, arr.n)), np.zeros(0), arr.lower, arr.upper, 0.0)


class Problem:
    """Instance with box primal set, orthant cone, optional dual ball."""

    def __init__(self, Q, q, r, A, b, lower, upper, mu=0.0):
        self.m = len(Q) - 1
        self.n = int(np.asarray(q[0]).shape[0])
        self.Q = [_storage(M, self.n) for M in Q]
        self.q = [np.asarray(v, dtype=float) for v in q]
        self.r = np.asarray(r, dtype=float)
        A = np.asarray(A.toarray() if sp.issparse(A) else A, dtype=float)
        self.p = A.shape[0] if A.size else int(np.asarray(b).shape[0])
        self.A = A.reshape(self.p, self.n)
        self.b = np.asarray(b, dtype=float).reshape(self.p)
        self.lo = np.asarray(lower, dtype=float)
        self.hi = np.asarray(upper, dtype=float)
        self.mu = float(mu)

    @classmethod
    def from_arrays(cls, arr):
        return cls(arr.Q_list(), arr.q_list(), arr.r, arr.A, arr.b,
                   arr.lower, arr.upper, arr.mu)

    # --- evaluations (problem.py:166-180) ---------------------------------
    def f(self, x):
        return 0.5 * float(x @ (self.Q[0] @ x)) + float(self.q[0] @ x) + self.r[0]

    def g(self, x):
        if self.m == 0:
            return np.zeros(0)
        vals = []
        for i in range(1, self.m + 1):
            vals.append(0.5 * float(x @ (self.Q[i] @ x)) + float(self.q[i] @ x) + self.r[i])
        return np.array(vals)

    def eq(self, x):
        return self.A @ x - self.b if self.p > 0 else np.zeros(0)

    def clip(self, w):
        return np.clip(w, self.lo, self.hi)

    # --- coupling (problem.py:196-223) -----------------------------------
    def phi(self, x, v, lam):
        val = self.f(x)
        if self.p > 0:
            val += float(v @ self.eq(x))
        if self.m > 0:
            val += float(lam @ self.g(x))
        return val

    def grad_x(self, x, v, lam):
        out = self.Q[0] @ x + self.q[0]
        for i in range(self.m):
            w = lam[i]
            if w != 0.0:
                out = out + w * (self.Q[i + 1] @ x + self.q[i + 1])
        if self.p > 0:
            out = out + self.A.T @ v
        return out


def half_sq_dist(a, b):
    """geometry.py:357-369 (Euclidean Bregman)."""
    d = np.asarray(a, dtype=float) - np.asarray(b, dtype=float)
    return 0.5 * float(d @ d)


class Ball:
    """Dual balls, geometry.py:263-311.  kind 0/1/2 = unbounded/joint/split."""

    def __init__(self, kind=0, r1=0.0, r2=0.0):
        self.kind, self.r1, self.r2 = kind, r1, r2

    def __call__(self, v, lam):
        if self.kind == 1:
            nrm = np.sqrt(v @ v + lam @ lam)
            if nrm <= self.r1:
                return v, lam
            s = self.r1 / nrm
            return s * v, s * lam
        if self.kind == 2:
            nv = np.linalg.norm(v)
            if nv > self.r1:
                v = (self.r1 / nv) * v
            nl = np.linalg.norm(lam)
            if nl > self.r2:
                lam = (self.r2 / nl) * lam
        return v, lam


@dataclass
class Options:
    """SolverConfig after resolved() (engine.py:33-63)."""
    mode: str = "yx"
    c_alpha: Optional[float] = None
    c_beta: Optional[float] = None
    delta: Optional[float] = None
    eta: float = 0.7
    tau_bar: float = 1.0
    gamma0: float = 1.0
    nonmonotone: bool = False
    ball: Ball = field(default_factory=Ball)
    max_backtracks: int = 200

    def resolve(self):
        d = {"xy": (0.25, 0.3, 0.4), "yx": (0.4, 0.0, 0.5)}[self.mode]
        if self.c_alpha is None:
            self.c_alpha = d[0]
        if self.c_beta is None:
            self.c_beta = d[1]
        if self.delta is None:
            self.delta = d[2]
        return self


@dataclass
class Row:
    """TraceRecord (engine.py:66-79)."""
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


class Engine:
    """engine.py:82-272 restated; state names follow the paper."""

    def __init__(self, P: Problem, opt: Options, x, v, lam, keep_iterates=False):
        self.P, self.o = P, opt.resolve()
        self.c_nm = 1.0 if opt.nonmonotone else 0.0
        self.iters = 0
        self.evals_total = 0
        self.trace: List[Row] = []
        self.iterates = []
        self.keep = keep_iterates
        self.reinit(x, v, lam)

    def reinit(self, x, v, lam, warm_tau=False):
        o, P = self.o, self.P
        x = P.clip(np.asarray(x, dtype=float))
        lam = np.maximum(np.asarray(lam, dtype=float), 0.0)
        v, lam = o.ball(np.asarray(v, dtype=float), lam)
        self.x, self.v, self.lam = x, v, lam
        t0 = self.tau_cand if (warm_tau and hasattr(self, "tau_cand")) else o.tau_bar
        self.tau_cand = t0
        self.tau_prev = t0
        self.gamma = o.gamma0
        self.sigma_prev = o.gamma0 * t0
        if o.mode == "xy":
            self.alpha = o.c_alpha / t0
            self.beta = o.c_beta / t0
            self.gx_cur = P.grad_x(x, v, lam)
            self.gx_prev = self.gx_cur.copy()
        else:
            self.alpha = o.c_alpha / self.sigma_prev
            self.beta = 0.0
            self.gy_cur = np.concatenate([P.eq(x), P.g(x)])
            self.gy_prev = self.gy_cur.copy()
        self.sigma0 = None
        self.x_cum = np.zeros(P.n)
        self.y_cum = np.zeros(P.p + P.m)
        self.T = 0.0

    @property
    def y(self):
        return np.concatenate([self.v, self.lam])

    def _trial_yx(self, tau, sigma):
        P, o = self.P, self.o
        theta = self.sigma_prev / sigma
        s = (1.0 + theta) * self.gy_cur - theta * self.gy_prev
        yt = self.y + sigma * s
        v_n = yt[:P.p]
        lam_n = np.maximum(yt[P.p:], 0.0)
        v_n, lam_n = o.ball(v_n, lam_n)
        gmix = P.grad_x(self.x, v_n, lam_n)
        x_n = P.clip(self.x - tau * gmix)
        gy_n = np.concatenate([P.eq(x_n), P.g(x_n)])
        # certificate (engine.py:151-163); gx at x_k recomputed as the reference does
        Dp = half_sq_dist(x_n, self.x)
        Dd = half_sq_dist(np.concatenate([v_n, lam_n]), self.y)
        g_at_k = P.grad_x(self.x, v_n, lam_n)
        lin = (P.phi(x_n, v_n, lam_n) - P.phi(self.x, v_n, lam_n)
               - float(g_at_k @ (x_n - self.x)))
        alpha_n = o.c_alpha / sigma
        E = (lin - Dp / tau
             + np.linalg.norm(gy_n - self.gy_cur) ** 2 / (2.0 * alpha_n)
             - (1.0 / sigma - theta * self.alpha) * Dd)
        return (x_n, v_n, lam_n), gy_n, E, Dp, Dd, alpha_n, 0.0

    def _trial_xy(self, tau, sigma):
        P, o = self.P, self.o
        theta = self.sigma_prev / sigma
        s = (1.0 + theta) * self.gx_cur - theta * self.gx_prev
        x_n = P.clip(self.x - tau * s)
        e_n, g_n = P.eq(x_n), P.g(x_n)
        v_n = self.v + sigma * e_n
        lam_n = np.maximum(self.lam + sigma * g_n, 0.0)
        v_n, lam_n = o.ball(v_n, lam_n)
        gx_yk = P.grad_x(x_n, self.v, self.lam)
        gx_n = P.grad_x(x_n, v_n, lam_n)
        alpha_n = o.c_alpha / tau
        beta_n = o.gamma0 * o.c_beta / sigma
        Dp = half_sq_dist(x_n, self.x)
        Dd = half_sq_dist(np.concatenate([v_n, lam_n]), self.y)
        E = (np.linalg.norm(gx_n - gx_yk) ** 2 / (2.0 * alpha_n)
             - Dd / sigma
             + np.linalg.norm(gx_yk - self.gx_cur) ** 2 / (2.0 * beta_n)
             - (1.0 / tau - theta * (self.alpha + self.beta)) * Dp)
        return (x_n, v_n, lam_n), gx_n, E, Dp, Dd, alpha_n, beta_n

    def step(self) -> Row:
        o, P = self.o, self.P
        tau = tau_start = self.tau_cand
        slack = 1e-13 * (1.0 + abs(P.phi(self.x, self.v, self.lam)))
        trial = self._trial_xy if o.mode == "xy" else self._trial_yx
        for count in range(1, o.max_backtracks + 2):
            sigma = self.gamma * tau
            z_n, cache_n, E, Dp, Dd, alpha_n, beta_n = trial(tau, sigma)
            if E <= -(o.delta / tau) * Dp - (o.delta / sigma) * Dd + slack:
                break
            tau *= o.eta
        else:
            raise OracleNonConvergence(
                "backtracking exhausted", {"tau": tau, "gamma": self.gamma, "iter": self.iters})
        evals = count
        g_next = self.gamma * (1.0 + P.mu * tau)
        tau_next = tau * np.sqrt((self.gamma / g_next) * (1.0 + self.c_nm * tau / self.tau_prev))
        if o.mode == "xy":
            self.gx_prev, self.gx_cur = self.gx_cur, cache_n
        else:
            self.gy_prev, self.gy_cur = self.gy_cur, cache_n
        self.x, self.v, self.lam = z_n
        self.alpha, self.beta = alpha_n, beta_n
        self.tau_prev, self.tau_cand = tau, tau_next
        self.sigma_prev = sigma
        self.gamma = g_next
        if self.sigma0 is None:
            self.sigma0 = sigma
        t_k = sigma / self.sigma0
        self.x_cum += t_k * self.x
        self.y_cum += t_k * np.concatenate([self.v, self.lam])
        self.T += t_k
        self.iters += 1
        self.evals_total += evals
        row = Row(self.iters, tau_start, tau, sigma, self.gamma, evals, self.evals_total)
        self.trace.append(row)
        if self.keep:
            self.iterates.append((self.x.copy(), self.v.copy(), self.lam.copy()))
        return row

    def last(self):
        return self.x, self.v, self.lam

    def average(self):
        if self.T <= 0:
            return self.last()
        xa = self.x_cum / self.T
        ya = self.y_cum / self.T
        return xa, ya[:self.P.p], ya[self.P.p:]


def initial_point(P: Problem, ball: Ball = None):
    """engine.py:275-283."""
    x = P.clip(np.zeros(P.n))
    lam = np.maximum(np.zeros(P.m), 0.0)
    v = np.zeros(P.p)
    if ball is not None:
        v, lam = ball(v, lam)
    return x, v, lam


# --- diagnostics -------------------------------------------------------------

@dataclass
class KKT:
    kkt_residual: float
    stationarity: float
    primal_eq: float
    complementarity: float
    infeas: float
    f_value: float
    mean_pos_violation: float
    subopt_abs: Optional[float] = None


def kkt(P: Problem, x, v, lam, f_star=None) -> KKT:
    """diagnostics.py:49-113 for the orthant cone."""
    gx = P.grad_x(x, v, lam)
    stat = float(np.linalg.norm(x - P.clip(x - gx)))
    eqn = float(np.linalg.norm(P.eq(x)))
    comp = float(np.linalg.norm(np.minimum(lam, -P.g(x)))) if P.m > 0 else 0.0
    fval = P.f(x)
    e = P.eq(x)
    gp = np.maximum(P.g(x), 0.0) if P.m > 0 else np.zeros(0)
    infeas = float(np.sqrt(e @ e + gp @ gp))
    mpv = float(np.mean(np.maximum(P.g(x), 0.0))) if P.m > 0 else 0.0
    return KKT(stat + eqn + comp, stat, eqn, comp, infeas, fval, mpv,
               None if f_star is None else fval - f_star)


def terminated(met: KKT, criterion="paper51", eps=1e-7, f_star=None,
               eps_kkt=1e-7, eps_feas=1e-7) -> bool:
    """diagnostics.py:252-263."""
    if criterion == "paper51":
        if f_star is None:
            return met.kkt_residual <= eps_kkt and met.infeas <= eps_feas
        rel = abs(met.f_value - f_star) / (1.0 + abs(f_star))
        return max(rel, met.mean_pos_violation) <= eps
    if criterion == "conic":
        return met.kkt_residual <= eps_kkt and met.infeas <= eps_feas
    raise OracleError(criterion)


def spectral_norm(M, iters=200, tol=1e-10):
    """problem.py:47-68."""
    rows, cols = M.shape
    if rows == 0 or cols == 0:
        return 0.0
    v = np.cos(np.arange(cols) + 0.5)
    v /= np.linalg.norm(v)
    prev = 0.0
    for _ in range(iters):
        w = M.T @ (M @ v)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            return 0.0
        v = w / nrm
        est = np.sqrt(nrm)
        done = abs(est - prev) <= tol * max(est, 1.0)
        prev = est
        if done:
            break
    return 1.01 * prev


def apg(value, grad, L, clip, x0, tol=1e-9, max_iter=50_000):
    """subsolve.py:27-62; returns (x, iterations, residual, converged)."""
    step = 1.0 / L
    x = clip(np.asarray(x0, dtype=float))
    yk = x.copy()
    t = 1.0
    fx = value(x)
    for it in range(1, max_iter + 1):
        xn = clip(yk - step * grad(yk))
        fn = value(xn)
        if fn > fx + 1e-12 * (1.0 + abs(fx)):
            xn = clip(x - step * grad(x))
            fn = value(xn)
            t = 1.0
        tn = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        yk = xn + ((t - 1.0) / tn) * (xn - x)
        x, fx, t = xn, fn, tn
        if it % 10 == 0 or it == max_iter:
            res = float(np.linalg.norm(x - clip(x - step * grad(x))))
            if res <= tol:
                return x, it, res, True
    res = float(np.linalg.norm(x - clip(x - step * grad(x))))
    return x, max_iter, res, res <= tol


def _dense(M):
    return M.toarray() if (sp.issparse(M) or hasattr(M, 'toarray')) else np.asarray(M)


def smoothed_gap(P: Problem, x, v, lam, xi, ball: Ball = None, tol=1e-9, x_warm=None):
    """diagnostics.py:120-163; returns (gap, (iterations, residual, converged))."""
    ball = ball or Ball()
    e, g = P.eq(x), P.g(x)
    v_h = v + e / (2.0 * xi)
    lam_h = np.maximum(lam + g / (2.0 * xi), 0.0)
    v_h, lam_h = ball(v_h, lam_h)
    dual_term = (P.phi(x, v_h, lam_h)
                 - 2.0 * xi * half_sq_dist(np.concatenate([v_h, lam_h]), np.concatenate([v, lam])))
    H = _dense(P.Q[0]).copy()
    for i in range(P.m):
        if lam[i] != 0.0:
            H = H + lam[i] * _dense(P.Q[i + 1])
    L = spectral_norm(H) + 2.0 * xi

    def value(xc):
        return P.phi(xc, v, lam) + 2.0 * xi * half_sq_dist(xc, x)

    def grad(xc):
        return P.grad_x(xc, v, lam) + 2.0 * xi * (xc - x)

    x0 = x if x_warm is None else x_warm
    xs, its, res, ok = apg(value, grad, L, P.clip, x0, tol=tol)
    return dual_term - value(xs), (its, res, ok)


# --- restart envelope (restarts.py:82-170) ------------------------------------

@dataclass
class Policy:
    kind: str = "none"          # none | fixed | adaptive
    period: int = 0
    xi: float = 0.04
    q: float = 0.5
    warmup: int = 50
    check_period: int = 200
    point: str = "last"


@dataclass
class Result:
    x: np.ndarray
    v: np.ndarray
    lam: np.ndarray
    avg: tuple
    trace: List[Row]
    restarts: list            # (outer, iteration, trigger, gap_new, gap_ref)
    iterations: int
    evals: int
    converged: bool
    status: str
    metrics: Optional[KKT]


def run_restarted(P: Problem, opt: Options, policy: Policy = None, z0=None,
                  budget=50_000, criteria: Optional[dict] = None, metrics_every=10,
                  warm_tau=False, on_iter=None) -> Result:
    """criteria: dict(criterion=, eps=, f_star=, eps_kkt=, eps_feas=) or None."""
    policy = policy or Policy()
    opt.resolve()
    if z0 is None:
        z0 = initial_point(P, opt.ball)
    eng = Engine(P, opt, *z0)
    log = []
    outer = inner = 0
    gap_ref = None
    x_warm = None
    converged, status, met = False, "budget", None
    f_star = criteria.get("f_star") if criteria else None

    def cand(kind):
        return eng.last() if kind == "last" else eng.average()

    for total in range(1, budget + 1):
        rec = eng.step()
        inner += 1
        if on_iter is not None:
            on_iter(total, eng)
        if criteria is not None and (total % metrics_every == 0 or total == budget):
            met = kkt(P, *eng.last(), f_star=f_star)
            rec.kkt, rec.infeas, rec.subopt = met.kkt_residual, met.infeas, met.subopt_abs
            if terminated(met, **criteria):
                converged, status = True, "converged"
                break
        if policy.kind == "fixed":
            if inner >= policy.period and total < budget:
                eng.reinit(*cand(policy.point), warm_tau=warm_tau)
                outer += 1
                inner = 0
                rec.restart_flag = 1
                log.append((outer, total, "fixed", None, None))
        elif policy.kind == "adaptive":
            due = ((gap_ref is None and total >= policy.warmup)
                   or (gap_ref is not None and inner >= policy.check_period
                       and inner % policy.check_period == 0))
            if due and total < budget:
                zc = cand(policy.point)
                tol = 1e-9 if gap_ref is None else min(1e-9, 0.01 * policy.xi * max(gap_ref, 0.0) + 1e-15)
                gap_new, _ = smoothed_gap(P, *zc, policy.xi, ball=opt.ball, tol=tol, x_warm=x_warm)
                x_warm = zc[0]
                rec.gap_xi = gap_new
                if gap_ref is None:
                    gap_ref = gap_new
                elif gap_new <= policy.q * gap_ref:
                    eng.reinit(*zc, warm_tau=warm_tau)
                    outer += 1
                    inner = 0
                    rec.restart_flag = 1
                    log.append((outer, total, "adaptive", gap_new, gap_ref))
                    gap_ref = gap_new
    if met is None:
        met = kkt(P, *eng.last(), f_star=f_star)
    return Result(eng.x, eng.v, eng.lam, eng.average(), eng.trace, log, eng.iters,
                  eng.evals_total, converged, status, met)
