"""Seeded synthetic instances for BASELINE.json configs C0-C4 (harness input).

Random source: the reference's counter generator "splitmix64-boxmuller/v1"
(``pkg/src/rapdb/rng.py:1-63``), restated so the same (seed, stream, index)
yields the same doubles on every platform.  Raw draw i of stream s under seed q
is ``mix(key + i)`` with ``key = mix(mix(q) + s)`` (``rng.py:35-45``); uniforms
take the top 53 bits (``rng.py:52-54``); normals are Box-Muller with the radius
from the first half of the raw draws and the angle from the second half
(``rng.py:56-63``) -- so normals are NOT call-granularity invariant and the call
sizes below are part of the contract.

Stream convention "4i..4i+3 for the i-th object" follows ``generate.py:51-61``.
Dense configs:

* ``B_i = normal(n*r) / sqrt(n)`` on stream 4i, C-order reshape to n x r;
* ``Q_i = 0.5*(M + M^T) + 0.1*I`` with ``M = B_i B_i^T`` (explicitly symmetrised);
* ``c_i = normal(n)`` on stream 4i+2;
* ``d_i = -uniform(1, 1, 2)`` on stream 4i+3 for i >= 1, ``d_0 = 0``;
* box [-10, 10]^n, orthant cone, no equalities.

Everything here builds host arrays once; they are fed unchanged to the device
path and to the CPU oracle.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

GENERATOR_NAME = "splitmix64-boxmuller/v1"

_M64 = 0xFFFFFFFFFFFFFFFF
_INC = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = 2.0 ** -53


def _finalize(z: np.ndarray) -> np.ndarray:
    """splitmix64 output function on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = z + _INC
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _mix_int(v: int) -> int:
    return int(_finalize(np.array([v & _M64], dtype=np.uint64))[0])


class CounterRng:
    """Stateless counter stream; each call consumes a contiguous index range."""

    name = GENERATOR_NAME

    def __init__(self, seed: int, stream: int = 0):
        self.key = np.uint64(_mix_int((_mix_int(seed) + stream) & _M64))
        self.counter = 0

    def raw(self, count: int) -> np.ndarray:
        idx = np.arange(self.counter, self.counter + count, dtype=np.uint64)
        self.counter += count
        with np.errstate(over="ignore"):
            return _finalize(idx + self.key)

    def uniform(self, count: int, low: float = 0.0, high: float = 1.0) -> np.ndarray:
        u = (self.raw(count) >> np.uint64(11)).astype(np.float64) * _TWO_M53
        return low + (high - low) * u

    def normal(self, count: int) -> np.ndarray:
        half = (count + 1) // 2
        bits = self.raw(2 * half) >> np.uint64(11)
        u1 = (bits[:half].astype(np.float64) + 1.0) * _TWO_M53
        u2 = bits[half:].astype(np.float64) * _TWO_M53
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 2.0 * np.pi * u2
        return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:count]


@dataclass
class QcqpArrays:
    """Plain host arrays of one instance.  ``Q`` is a C-contiguous
    ``(m+1, n, n)`` stack (index 0 = objective), ``q`` is ``(m+1, n)``."""

    n: int
    m: int
    p: int
    Q: np.ndarray
    q: np.ndarray
    r: np.ndarray
    A: np.ndarray
    b: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    mu: float = 0.0
    name: str = ""
    meta: dict = field(default_factory=dict)

    def Q_list(self) -> List[np.ndarray]:
        return [self.Q[i] for i in range(self.m + 1)]

    def q_list(self) -> List[np.ndarray]:
        return [self.q[i] for i in range(self.m + 1)]


def dense_qcqp(n: int, m: int, rank: int, seed: int = 0,
               box: float = 10.0) -> QcqpArrays:
    """BASELINE configs 0-2: ``Q_i = B_i B_i^T + 0.1 I`` (i = 0..m)."""
    Q = np.empty((m + 1, n, n), dtype=np.float64)
    q = np.empty((m + 1, n), dtype=np.float64)
    r = np.zeros(m + 1, dtype=np.float64)
    scale = 1.0 / np.sqrt(n)
    for i in range(m + 1):
        B = CounterRng(seed, 4 * i).normal(n * rank).reshape(n, rank) * scale
        M = B @ B.T
        Qi = Q[i]
        np.add(M, M.T, out=Qi)
        Qi *= 0.5
        Qi[np.diag_indices(n)] += 0.1
        q[i] = CounterRng(seed, 4 * i + 2).normal(n)
        if i > 0:
            r[i] = -float(CounterRng(seed, 4 * i + 3).uniform(1, 1.0, 2.0)[0])
    return QcqpArrays(
        n=n, m=m, p=0, Q=Q, q=q, r=r,
        A=np.zeros((0, n)), b=np.zeros(0),
        lower=np.full(n, -box), upper=np.full(n, box), mu=0.0,
        name=f"dense-qcqp-n{n}-m{m}-r{rank}-s{seed}",
        meta={"generator": GENERATOR_NAME, "seed": seed, "rank": rank})


def kml_epigraph(N: int = 4000, d: int = 50, seed: int = 0,
                 C: float = 1.0) -> QcqpArrays:
    """BASELINE config 4: kernel-matrix-learning QCQP in epigraph form.

    Points: ``a_k = y_k*0.5*1 + N(0, I_d)`` (normals on stream 0, N*d draws),
    balanced labels (first half +1).  Kernels: RBF with widths
    {0.1, 1, 10} x median pairwise distance (``exp(-|a-a'|^2/(2w^2))``),
    ``(1 + a.a')^2`` and ``a.a'``; each scaled to trace N.  ``Q_j = diag(y) K_j
    diag(y)``.  Variables ``(alpha, t)``, n = N+1; minimise t subject to
    ``(1/N) alpha^T Q_j alpha - 2 1^T alpha - t <= 0``, i.e. ``Qt_j = (2/N) Q_j
    (+) 0``, ``q_j = (-2*1, -1)``, ``r_j = 0``; ``y^T alpha = 0`` (p = 1);
    ``0 <= alpha <= C``, t free.  Objective f = t (``Q_0 = 0``, ``q_0 = e_t``).
    """
    rng = CounterRng(seed, 0)
    y = np.concatenate([np.ones(N // 2), -np.ones(N - N // 2)])
    X = rng.normal(N * d).reshape(N, d) + 0.5 * y[:, None]
    G = X @ X.T
    sq = np.diag(G).copy()
    D2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * G, 0.0)
    iu = np.triu_indices(N, 1)
    med = float(np.median(np.sqrt(D2[iu])))
    kernels = []
    for wmul in (0.1, 1.0, 10.0):
        w = wmul * med
        kernels.append(np.exp(-D2 / (2.0 * w * w)))
    kernels.append((1.0 + G) ** 2)
    kernels.append(G.copy())
    n = N + 1
    m = len(kernels)
    Q = np.zeros((m + 1, n, n), dtype=np.float64)
    q = np.zeros((m + 1, n), dtype=np.float64)
    q[0, N] = 1.0
    yy = np.outer(y, y)
    for j, K in enumerate(kernels):
        K = K * (N / np.trace(K))
        H = yy * K
        H = 0.5 * (H + H.T)
        Q[j + 1, :N, :N] = (2.0 / N) * H
        q[j + 1, :N] = -2.0
        q[j + 1, N] = -1.0
    A = np.zeros((1, n))
    A[0, :N] = y
    lower = np.zeros(n)
    upper = np.full(n, C)
    lower[N] = -np.inf
    upper[N] = np.inf
    return QcqpArrays(
        n=n, m=m, p=1, Q=Q, q=q, r=np.zeros(m + 1), A=A, b=np.zeros(1),
        lower=lower, upper=upper, mu=0.0, name=f"kml-epigraph-N{N}-d{d}-s{seed}",
        meta={"generator": GENERATOR_NAME, "seed": seed, "median_dist": med})


@dataclass
class FactoredArrays:
    """Config-3 style instance: Q_i = R_i^T R_i (i = 0..mq, i = 0 objective) with
    the R_i stacked into one CSR ``R`` (row block i = rows [i*r, (i+1)*r)), dense
    linear terms ``C [mq+1][n]``, constants ``d``, and a sparse linear block
    ``A x <= b`` treated as orthant constraints with Q = 0 (so the constraint
    vector is (g_1..g_mq, A x - b))."""

    n: int
    mq: int
    rows: int                  # rows per R_i
    R: object                  # scipy.sparse.csr_matrix ((mq+1)*rows, n)
    C: np.ndarray              # (mq+1, n)
    d: np.ndarray              # (mq+1,)
    A: object                  # scipy.sparse.csr_matrix (L, n)
    b: np.ndarray              # (L,)
    lower: np.ndarray
    upper: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:        # total constraints: quadratic + linear rows
        return self.mq + self.A.shape[0]

    @property
    def L(self) -> int:        # linear inequality rows
        return self.A.shape[0]

    def block(self, i: int):
        """R_i (CSR rows [i*rows, (i+1)*rows) of the stack)."""
        return self.R[i * self.rows:(i + 1) * self.rows]

    def dense_lists(self):
        """(Q list, q list, r) as the reference's ProblemInstance holds this
        instance: dense Q_i = R_i^T R_i (its ``_as_operator`` turns them into CSR
        when sparse enough, problem.py:31-40), zero Q for each linear row
        (problem.py:38-39), q = (c_0..c_mq, a_1..a_L), r = (d_0..d_mq, -b).
        Small instances only (m+1 dense n x n matrices)."""
        Q = [np.asarray((self.block(i).T @ self.block(i)).toarray()) for i in range(self.mq + 1)]
        Q += [np.zeros((self.n, self.n)) for _ in range(self.L)]
        Ad = self.A.toarray()
        q = [self.C[i].copy() for i in range(self.mq + 1)] + [Ad[j].copy() for j in range(self.L)]
        r = np.concatenate([self.d, -self.b])
        return Q, q, r


def _csr_uniform(rng_vals, rng_cols, nrows, ncols, nnz_row, scale):
    import scipy.sparse as sp
    vals = rng_vals.normal(nrows * nnz_row) * scale
    cols = np.minimum((rng_cols.uniform(nrows * nnz_row) * ncols).astype(np.int64), ncols - 1)
    indptr = np.arange(0, nrows * nnz_row + 1, nnz_row, dtype=np.int64)
    return sp.csr_matrix((vals, cols, indptr), shape=(nrows, ncols))


def factored_qcqp(n: int = 1_000_000, mq: int = 64, rows: int = 100_000, nnz_row: int = 10,
                  lin_rows: int = 500_000, lin_nnz: int = 5, seed: int = 0, box: float = 10.0,
                  x0_scale: float = 1.0) -> FactoredArrays:
    """BASELINE config 3 (defaults = full size).  Streams: R_i values on 4i
    (N(0,1)/sqrt(nnz_row)), columns on 4i+1 (uniform), c_i on 4i+2
    (N(0,1)/sqrt(n)), d_i = -U(1,2) on 4i+3 (d_0 = 0).  Linear block: values on
    4(mq+1) (N(0,1)), columns on 4(mq+1)+1, x0 ~ U(-1,1) on 4(mq+1)+2,
    b = A x0 + U(0,1) on 4(mq+1)+3.  Q_0 = R_0^T R_0 is an assumption (the
    BASELINE text leaves the objective unspecified).
    ``x0_scale`` shrinks x0 (parity cases use 0.2 so that x0 is strictly
    feasible for the quadratic rows too; BASELINE's own text has 1)."""
    import scipy.sparse as sp
    blocks, C, d = [], np.empty((mq + 1, n)), np.zeros(mq + 1)
    for i in range(mq + 1):
        blocks.append(_csr_uniform(CounterRng(seed, 4 * i), CounterRng(seed, 4 * i + 1), rows, n, nnz_row,
                                   1.0 / np.sqrt(nnz_row)))
        C[i] = CounterRng(seed, 4 * i + 2).normal(n) / np.sqrt(n)
        if i > 0:
            d[i] = -float(CounterRng(seed, 4 * i + 3).uniform(1, 1.0, 2.0)[0])
    R = sp.vstack(blocks, format="csr")
    s = 4 * (mq + 1)
    A = _csr_uniform(CounterRng(seed, s), CounterRng(seed, s + 1), lin_rows, n, lin_nnz, 1.0)
    x0 = CounterRng(seed, s + 2).uniform(n, -1.0, 1.0) * x0_scale
    b = A @ x0 + CounterRng(seed, s + 3).uniform(lin_rows, 0.0, 1.0)
    return FactoredArrays(n=n, mq=mq, rows=rows, R=R, C=C, d=d, A=A, b=b,
                          lower=np.full(n, -box), upper=np.full(n, box),
                          name=f"factored-qcqp-n{n}-m{mq}-r{rows}-L{lin_rows}-s{seed}",
                          meta={"generator": GENERATOR_NAME, "seed": seed, "nnz_row": nnz_row,
                                "lin_nnz": lin_nnz})


def sparse_qcqp(n: int = 400, m: int = 6, rows: int = 60, nnz_row: int = 4, seed: int = 0, box: float = 10.0):
    """A QCQP with SPARSE quadratic forms (below the reference's 25 % CSR
    limit, problem.py:31-40): Q_i = B_i^T B_i + 0.1 I with B_i [rows x n],
    nnz_row entries per row (the streams of factored_qcqp), q_i ~ N(0,1)/sqrt(n),
    r_i = -U(1,2) (r_0 = 0), box [-box, box].  Returns (Q list of CSR with
    sorted indices, q [(m+1) x n], r [m+1], lower, upper)."""
    import scipy.sparse as sp
    Q, q, r = [], np.empty((m + 1, n)), np.zeros(m + 1)
    for i in range(m + 1):
        B = _csr_uniform(CounterRng(seed, 4 * i), CounterRng(seed, 4 * i + 1), rows, n, nnz_row,
                         1.0 / np.sqrt(nnz_row))
        M = (B.T @ B + 0.1 * sp.identity(n, format="csr")).tocsr()
        M = ((M + M.T) * 0.5).tocsr()
        M.sum_duplicates()
        M.sort_indices()
        Q.append(M)
        q[i] = CounterRng(seed, 4 * i + 2).normal(n) / np.sqrt(n)
        if i > 0:
            r[i] = -float(CounterRng(seed, 4 * i + 3).uniform(1, 1.0, 2.0)[0])
    return Q, q, r, np.full(n, -box), np.full(n, box)


# BASELINE.json configs[0..2], [4]; config 3 (factored sparse) is factored_qcqp()
CONFIGS = {
    "C0": dict(n=200, m=10, rank=20),
    "C1": dict(n=2000, m=200, rank=200),
    "C2": dict(n=4096, m=512, rank=256),
}


def config_instance(name: str, seed: int = 0, scale: Optional[float] = None) -> QcqpArrays:
    """Instance for a BASELINE config name; ``scale`` shrinks n and m
    proportionally (parity cases at sizes the oracle finishes quickly)."""
    if name == "C4":
        N = 4000 if scale is None else max(8, int(4000 * scale))
        return kml_epigraph(N=N)
    cfg = dict(CONFIGS[name])
    if scale is not None:
        cfg = dict(n=max(4, int(cfg["n"] * scale)), m=max(1, int(cfg["m"] * scale)),
                   rank=max(2, int(cfg["rank"] * scale)))
    return dense_qcqp(seed=seed, **cfg)
