"""QCQP instances, iterates and the coupling-function operator contract.

Mirrors ``pkg/src/rapdb/problem.py`` (``ProblemInstance`` :109-162, ``Iterate``
:71-89, ``coupling_value``/``grad_x_coupling``/``grad_y_coupling`` :196-223) for
the hot path's instance class: dense Q_i, box primal set, nonnegative-orthant
cone, optional equality block ``Ax = b``.

Storage differs from the reference by design: instead of
a Python list of m+1 dense arrays / CSR matrices (``_as_operator``
:31-40), the device holds ONE contiguous fp64 stack ``[m+1][n][ld]`` (ld = n
rounded up to even so every row is a 16-byte-aligned bulk-copy source) and the
solver streams it once per test evaluation.  ``DeviceData`` is that upload.

The operator-contract functions evaluate on the GPU (one probe sweep + a few
device vector ops); nothing here evaluates Q products on the host.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import ConfigurationError, DeviceError, InputError
from .geometry import Box, NonnegOrthant, cone_dim, set_dim


@dataclass(frozen=True)
class Iterate:
    """Primal-dual point z = (x, v, lam)."""

    x: np.ndarray
    v: np.ndarray
    lam: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "x", np.asarray(self.x, dtype=float))
        object.__setattr__(self, "v", np.asarray(self.v, dtype=float))
        object.__setattr__(self, "lam", np.asarray(self.lam, dtype=float))

    @property
    def y(self):
        return np.concatenate([self.v, self.lam])

    def dual_norm(self) -> float:
        return float(np.sqrt(self.v @ self.v + self.lam @ self.lam))


def _dense(M):
    return M.toarray() if hasattr(M, "toarray") else np.asarray(M, dtype=float)


@dataclass(frozen=True)
class ProblemInstance:
    """Immutable QCQP data; Q[0] is the objective, Q[1..m] the constraints.

    ``Q`` may be a list of m+1 (n, n) arrays (reference style) or one
    C-contiguous ``(m+1, n, n)`` float64 stack (no copy is made).  ``validate``
    mirrors the reference's load-time checks (problem.py:142-162: symmetry to
    1e-12, lambda_min >= -1e-10, rank(A) = p); pass ``validate=False`` for the
    multi-GB benchmark instances whose generators guarantee both.
    """

    n: int
    m: int
    p: int
    Q: object
    q: object
    r: np.ndarray
    A: object
    b: np.ndarray
    primal_set: Box
    cone: NonnegOrthant
    mu: float = 0.0
    dual_set: Optional[object] = None
    name: str = ""
    validate: bool = field(default=True, compare=False)

    def __post_init__(self):
        n, m, p = self.n, self.m, self.p
        if n <= 0 or m < 0 or p < 0:
            raise InputError("need n > 0, m >= 0, p >= 0")
        Q = self.Q
        if isinstance(Q, np.ndarray) and Q.ndim == 3:
            if Q.shape != (m + 1, n, n):
                raise InputError("need m+1 quadratic forms (objective plus m constraints)")
            stack = np.ascontiguousarray(Q, dtype=np.float64)
        else:
            if len(Q) != m + 1:
                raise InputError("need m+1 quadratic forms (objective plus m constraints)")
            mats = [_dense(M) for M in Q]
            for i, M in enumerate(mats):
                if M.shape != (n, n):
                    raise InputError(f"quadratic form {i} has wrong dimensions")
            stack = np.ascontiguousarray(np.stack(mats), dtype=np.float64)
        if isinstance(self.q, (list, tuple)):
            qa = (np.stack([np.asarray(v, dtype=float) for v in self.q]) if len(self.q)
                  else np.zeros((0, n)))
        else:
            qa = np.asarray(self.q, dtype=float)
        if qa.shape != (m + 1, n):
            raise InputError("need m+1 linear terms of length n")
        r = np.asarray(self.r, dtype=float)
        if r.shape != (m + 1,):
            raise InputError("need m+1 constants")
        A = np.asarray(_dense(self.A) if p else np.zeros((0, n)), dtype=float).reshape(p, n)
        b = np.asarray(self.b, dtype=float).reshape(p)
        object.__setattr__(self, "Q", stack)
        object.__setattr__(self, "q", np.ascontiguousarray(qa))
        object.__setattr__(self, "r", r)
        object.__setattr__(self, "A", np.ascontiguousarray(A))
        object.__setattr__(self, "b", b)
        if set_dim(self.primal_set) != n:
            raise InputError("primal set dimension mismatch")
        if cone_dim(self.cone) != m:
            raise InputError("cone dimension mismatch")
        if self.mu < 0:
            raise InputError("strong convexity modulus must be nonnegative")
        if self.validate:
            for i in range(m + 1):
                D = stack[i]
                if np.max(np.abs(D - D.T)) > 1e-12 * max(1.0, np.max(np.abs(D))):
                    raise InputError(f"Q[{i}] is not symmetric")
                lam_min = float(np.linalg.eigvalsh(D)[0])
                if lam_min < -1e-10:
                    raise InputError(f"Q[{i}] has negative eigenvalue {lam_min:.3e}")
            if p > 0 and np.linalg.matrix_rank(A) < p:
                raise InputError("equality matrix A is not full row rank")
            if self.mu > 0:
                lam0 = float(np.linalg.eigvalsh(stack[0])[0])
                if self.mu > lam0 + 1e-10:
                    raise InputError(f"declared mu={self.mu} exceeds lambda_min(Q0)={lam0:.3e}")
        object.__setattr__(self, "_dev", {})

    @classmethod
    def from_arrays(cls, arr, validate=True):
        """From ``instances.QcqpArrays``."""
        return cls(n=arr.n, m=arr.m, p=arr.p, Q=arr.Q, q=arr.q, r=arr.r, A=arr.A, b=arr.b,
                   primal_set=Box(arr.lower, arr.upper), cone=NonnegOrthant(arr.m), mu=arr.mu,
                   name=arr.name, validate=validate)

    def check_device_support(self):
        if self.dual_set is not None:
            raise ConfigurationError("minimax dual_set instances are not built on the device path")
        if not isinstance(self.primal_set, Box):
            raise ConfigurationError("the device path supports Box primal sets")
        if not isinstance(self.cone, NonnegOrthant):
            raise ConfigurationError("the device path supports the nonnegative orthant cone")

    def device_data(self, device=None, pinned_host=None, krange=None):
        """Upload (cached per device and matrix range).  ``pinned_host``: optional
        pinned torch copy of the Q stack; ``krange=(k0, k1)``: upload only the
        matrices of one constraint shard."""
        import torch
        dev = torch.device("cuda", 0) if device is None else torch.device(device)
        k0, k1 = krange if krange is not None else (0, self.m + 1)
        key = str(dev) if (k0, k1) == (0, self.m + 1) else f"{dev}[{k0}:{k1}]"
        cache = self._dev
        if key not in cache:
            src = pinned_host if pinned_host is not None else cache.get("_pinned")
            cache[key] = DeviceData.upload(self, dev, src, k0, k1)
        return cache[key]

    def zero_flags(self) -> np.ndarray:
        """All-zero flags of the m+1 matrices (computed once: the instance is
        immutable).  All-zero matrices are never streamed (C4's Q_0)."""
        z = self._dev.get("_zero")
        if z is None:
            z = np.array([not np.any(self.Q[i]) for i in range(self.m + 1)], dtype=np.uint8)
            self._dev["_zero"] = z
        return z

    def pin_host(self):
        """Keep a page-locked copy of the Q stack so uploads run at full PCIe rate."""
        import torch
        if "_pinned" not in self._dev:
            self._dev["_pinned"] = torch.from_numpy(self.Q).pin_memory()
        return self._dev["_pinned"]

    def drop_device_data(self):
        """Release the device copies (the pinned host copy and zero flags are kept)."""
        for k in [k for k in self._dev if k not in ("_pinned", "_zero")]:
            del self._dev[k]

    # -- evaluations (problem.py:166-186) on the device --------------------
    def _evaluator(self):
        from .engine import _Evaluator
        ev = self._dev.get("_eval")
        if ev is None:
            ev = _Evaluator(self)
            self._dev["_eval"] = ev
        return ev

    def f_value(self, x) -> float:
        return float(self._evaluator().sweep(x)[1][0])

    def g_value(self, x) -> np.ndarray:
        if self.m == 0:
            return np.zeros(0)
        return self._evaluator().sweep(x)[1][1:].cpu().numpy()

    def eq_residual(self, x) -> np.ndarray:
        if self.p == 0:
            return np.zeros(0)
        return self._evaluator().eq(x).cpu().numpy()

    def project_dual_cone(self, lam):
        return np.maximum(np.asarray(lam, dtype=float), 0.0)


class DeviceData:
    """The instance resident in HBM: Q stack [m+1][n][ld] + vectors (fp64)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @classmethod
    def upload(cls, inst: ProblemInstance, device, pinned_host=None, k0=0, k1=None, layout=None):
        """layout "packed" (default; env RAPDB_LAYOUT): the upper block
        triangle in 32 x 32 sub-tiles (csrc/symsweep.cuh), half the bytes of
        the stack; "rows": the row-major stack [k1-k0][n][ld]."""
        import torch
        n, m, p = inst.n, inst.m, inst.p
        k1 = m + 1 if k1 is None else k1
        ld = n + (n & 1)
        layout = layout or os.environ.get("RAPDB_LAYOUT", "packed")
        if layout not in ("packed", "rows"):
            raise ConfigurationError(f"unknown Q-stack layout {layout!r}")
        zero = inst.zero_flags()[k0:k1].copy()
        src = (pinned_host if pinned_host is not None else torch.from_numpy(inst.Q))[k0:k1]
        if layout == "packed":
            Qd = _upload_packed(src, n, device, pinned_host is not None)
        elif ld == n:
            Qd = src.to(device, non_blocking=pinned_host is not None)
        else:
            Qd = torch.zeros((k1 - k0, n, ld), dtype=torch.float64, device=device)
            Qd[:, :, :n].copy_(src, non_blocking=pinned_host is not None)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)
        lo = inst.primal_set.lower
        hi = inst.primal_set.upper
        return cls(n=n, m=m, p=p, ld=ld, Q=Qd, q=t(inst.q), r=t(inst.r),
                   A=t(inst.A) if p else None, b=t(inst.b) if p else None,
                   lower=t(lo), upper=t(hi), mu=float(inst.mu), zero_flags=zero, device=device,
                   layout=layout)


def packed_source_elements(n: int) -> int:
    """Entries of one dense n x n matrix that the packed layout stores (and that
    a pack straight from page-locked host memory reads over PCIe): the upper
    32-block triangle, diagonal 64-units without their (1,0) sub-tile."""
    nb32 = (n + 31) // 32
    ext = [min(32, n - 32 * k) for k in range(nb32)]
    tot = 0
    for bi in range(nb32):
        for bj in range(bi, nb32):
            tot += ext[bi] * ext[bj]
    return tot


def _upload_packed(src, n, device, pinned):
    """Dense host matrices -> packed symmetric stack on the device.  Page-locked
    sources are packed straight from host memory (only the upper triangle
    crosses PCIe; env RAPDB_PACK_STAGED=1 forces staging); otherwise chunks
    of <= 1 GB are staged on the device and packed there."""
    import torch
    from . import _capi
    cnt = src.shape[0]
    spm = _capi.packed_doubles(n)
    Qp = torch.empty((max(cnt, 1), spm), dtype=torch.float64, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    if cnt == 0:
        return Qp
    if pinned and os.environ.get("RAPDB_PACK_STAGED", "0") != "1":
        _capi.pack_symmetric(n, cnt, src.data_ptr(), n, n * n, Qp.data_ptr(), stream)
        return Qp
    chunk = max(1, min(cnt, (1 << 30) // (n * n * 8)))
    stage = torch.empty((chunk, n, n), dtype=torch.float64, device=device)
    for c0 in range(0, cnt, chunk):
        c = min(chunk, cnt - c0)
        stage[:c].copy_(src[c0:c0 + c], non_blocking=pinned)
        _capi.pack_symmetric(n, c, stage.data_ptr(), n, n * n, Qp[c0].data_ptr(), stream)
    del stage
    return Qp


@dataclass
class LipschitzConstants:
    """Same fields as the reference's (problem.py:93-106).  The constants are
    only used for the reference's analysis and stepsize heuristics outside the
    hot path (out of scope); compute_constants raises."""

    L_f: float
    L_g: float
    B_g: float
    C_g: float
    L_xx: float
    L_xy: float
    Lhat_xx: float
    Lhat_yx: float
    dual_bound_used: float
    psi1: float
    psi2: float
    B_g_is_estimate: bool = False
    bar_B_used: float = np.inf


def spectral_norm(M, iters: int = 200, tol: float = 1e-10, device=None) -> float:
    """problem.py:47-68 on the device (rapdb_spectral_norm): power iteration on
    M'M from cos(k + 1/2), stop when |est - prev| <= tol max(est, 1), 1.01
    inflation.  Sparse M is densified for the device product."""
    import torch
    from . import _capi
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: spectral_norm runs on the GPU (no CPU fallback)")
    Md = M.toarray() if hasattr(M, "toarray") else np.asarray(M, dtype=np.float64)
    Md = np.ascontiguousarray(Md, dtype=np.float64)
    if Md.ndim != 2:
        raise InputError("spectral_norm needs a matrix")
    if Md.shape[0] == 0 or Md.shape[1] == 0:
        return 0.0
    dev = torch.device("cuda", 0) if device is None else torch.device(device)
    return _capi.spectral_norm(torch.from_numpy(Md).to(dev), iters, tol)


def compute_constants(*args, **kwargs):
    """problem.py:226-317 of the reference (Lipschitz constants and dual
    bounds for the analysis): not part of the device hot path."""
    raise ConfigurationError("compute_constants (problem.py:226-317) is outside the B200 hot path; "
                             "use the reference package for the analysis constants")


def _check_point(inst: ProblemInstance, z: Iterate):
    if z.x.shape != (inst.n,) or z.v.shape != (inst.p,) or z.lam.shape != (inst.m,):
        raise InputError(
            f"iterate dims {(z.x.shape, z.v.shape, z.lam.shape)} do not match "
            f"instance (n={inst.n}, p={inst.p}, m={inst.m})")


def coupling_value(inst: ProblemInstance, z: Iterate) -> float:
    """Phi(x, y) = f(x) + v'(Ax - b) + lam'g(x) (problem.py:196-204), on device."""
    _check_point(inst, z)
    return inst._evaluator().coupling(z)


def grad_x_coupling(inst: ProblemInstance, z: Iterate) -> np.ndarray:
    """(Q0 + sum lam_i Q_i) x + q0 + sum lam_i q_i + A'v (problem.py:207-217), on device."""
    _check_point(inst, z)
    return inst._evaluator().grad_x(z)


def grad_y_coupling(inst: ProblemInstance, z: Iterate):
    """(Ax - b, g(x)) (problem.py:220-223), on device."""
    _check_point(inst, z)
    return inst.eq_residual(z.x), inst.g_value(z.x)


class DeviceDenseInstance:
    """A dense QCQP of BASELINE configs 0-2's family whose Q stack is generated
    ON THE DEVICE and packed there (never materialised on the host):
    ``Q_i = 0.5 (B_i B_i^T + (B_i B_i^T)^T) + 0.1 I`` with ``B_i`` of shape n x r
    and N(0, 1)/sqrt(n) entries drawn by torch's CUDA generator seeded with
    (seed, i), fp64 DGEMM on the device; ``c_i ~ N(0,1)``, ``d_i ~ -U(1, 2)``,
    ``d_0 = 0``, box [-box, box]^n, orthant cone, no equalities.  Same
    distribution as ``instances.dense_qcqp`` but a different random stream (the
    CounterRng instances stay the parity inputs); used for C2-scale
    throughput runs, where the host instance would need 69 GB of host RAM.
    Each rank of a sharded run generates only its own matrices.  Exposes the
    ``ProblemInstance`` surface the solver layers use."""

    def __init__(self, n: int, m: int, rank: int, seed: int = 0, box: float = 10.0, name: str = ""):
        self.n, self.m, self.p, self.rank_r, self.seed = int(n), int(m), 0, int(rank), int(seed)
        rng = np.random.default_rng(seed)
        self.q = rng.standard_normal((m + 1, n))
        self.r = np.concatenate([[0.0], -rng.uniform(1.0, 2.0, m)])
        self.A = np.zeros((0, n))
        self.b = np.zeros(0)
        self.mu = 0.0
        self.dual_set = None
        self.name = name or f"device-dense n={n} m={m} r={rank}"
        self.meta = {"rank": int(rank), "seed": int(seed), "generator": "torch CUDA normal + fp64 DGEMM"}
        self.primal_set = Box(np.full(n, -box), np.full(n, box))
        self.cone = NonnegOrthant(m)
        self._dev = {}

    def check_device_support(self):
        return None

    def zero_flags(self) -> np.ndarray:
        return np.zeros(self.m + 1, dtype=np.uint8)

    def generate_packed(self, device, k0: int, k1: int):
        import torch
        from . import _capi
        n, r = self.n, self.rank_r
        cnt = k1 - k0
        spm = _capi.packed_doubles(n)
        Qp = torch.empty((max(cnt, 1), spm), dtype=torch.float64, device=device)
        chunk = max(1, min(cnt, (1 << 30) // (n * n * 8)))
        stage = torch.empty((chunk, n, n), dtype=torch.float64, device=device)
        gen = torch.Generator(device=device)
        stream = torch.cuda.current_stream(device).cuda_stream
        eye = 0.1 * torch.eye(n, dtype=torch.float64, device=device)
        for c0 in range(0, cnt, chunk):
            c = min(chunk, cnt - c0)
            for j in range(c):
                gen.manual_seed(self.seed * 1_000_003 + k0 + c0 + j)
                B = torch.randn((n, r), generator=gen, dtype=torch.float64, device=device) / np.sqrt(n)
                M = B @ B.T
                stage[j] = 0.5 * (M + M.T) + eye
            _capi.pack_symmetric(n, c, stage.data_ptr(), n, n * n, Qp[c0].data_ptr(), stream)
        del stage
        return Qp

    def device_data(self, device=None, pinned_host=None, krange=None):
        import torch
        dev = torch.device("cuda", 0) if device is None else torch.device(device)
        k0, k1 = krange if krange is not None else (0, self.m + 1)
        key = str(dev) if (k0, k1) == (0, self.m + 1) else f"{dev}[{k0}:{k1}]"
        if key not in self._dev:
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
            n = self.n
            self._dev[key] = DeviceData(n=n, m=self.m, p=0, ld=n + (n & 1), Q=self.generate_packed(dev, k0, k1),
                                        q=t(self.q), r=t(self.r), A=None, b=None,
                                        lower=t(self.primal_set.lower), upper=t(self.primal_set.upper), mu=0.0,
                                        zero_flags=np.zeros(k1 - k0, dtype=np.uint8), device=dev,
                                        layout="packed")
        return self._dev[key]

    def drop_device_data(self):
        self._dev.clear()

    def _evaluator(self):
        from .engine import _Evaluator
        ev = self._dev.get("_eval")
        if ev is None:
            ev = _Evaluator(self)
            self._dev["_eval"] = ev
        return ev

    def f_value(self, x) -> float:
        return float(self._evaluator().sweep(x)[1][0])

    def g_value(self, x) -> np.ndarray:
        return self._evaluator().sweep(x)[1][1:].cpu().numpy()

    def eq_residual(self, x) -> np.ndarray:
        return np.zeros(0)

    def project_dual_cone(self, lam):
        return np.maximum(np.asarray(lam, dtype=float), 0.0)


# ---------------------------------------------------------------------------
# The reference's problem JSON (problem.py:318-389): dense matrices as nested
# lists, sparse ones as {"format": "csr", ...}; sets and cones as descriptors.

def _matrix_to_json(M):
    M = np.asarray(M)
    if M.ndim == 2 and M.size and np.count_nonzero(M) < 0.25 * M.size:
        import scipy.sparse as sp
        S = sp.csr_matrix(M)
        return {"format": "csr", "shape": list(S.shape), "indptr": S.indptr.tolist(),
                "indices": S.indices.tolist(), "data": S.data.tolist()}
    return M.tolist()


def _matrix_from_json(obj, shape):
    if isinstance(obj, dict):
        if obj.get("format") != "csr":
            raise InputError(f"unknown matrix format {obj.get('format')!r}")
        import scipy.sparse as sp
        return sp.csr_matrix((obj["data"], obj["indices"], obj["indptr"]),
                             shape=tuple(obj.get("shape", shape))).toarray()
    return np.asarray(obj, dtype=float).reshape(shape)


def to_json_dict(inst: ProblemInstance) -> dict:
    from .geometry import cone_to_json, set_to_json
    out = {
        "n": inst.n, "m": inst.m, "p": inst.p,
        "Q": [_matrix_to_json(inst.Q[i]) for i in range(inst.m + 1)],
        "q": [v.tolist() for v in inst.q],
        "r": inst.r.tolist(),
        "A": np.asarray(inst.A).tolist(),
        "b": inst.b.tolist(),
        "primal_set": set_to_json(inst.primal_set),
        "cone": cone_to_json(inst.cone),
        "mu": inst.mu,
    }
    if inst.name:
        out["name"] = inst.name
    return out


def from_json_dict(d: dict, validate: bool = True) -> ProblemInstance:
    from .geometry import cone_from_json, set_from_json
    if "dual_set" in d:
        raise ConfigurationError("minimax dual_set instances are not built on the device path")
    try:
        n, m, p = int(d["n"]), int(d["m"]), int(d["p"])
        return ProblemInstance(
            n=n, m=m, p=p,
            Q=[_matrix_from_json(M, (n, n)) for M in d["Q"]],
            q=[np.asarray(v, dtype=float) for v in d["q"]],
            r=np.asarray(d["r"], dtype=float),
            A=np.asarray(d["A"], dtype=float).reshape(p, n),
            b=np.asarray(d["b"], dtype=float),
            primal_set=set_from_json(d["primal_set"]),
            cone=cone_from_json(d["cone"]),
            mu=float(d.get("mu", 0.0)),
            name=str(d.get("name", "")),
            validate=validate)
    except (KeyError, TypeError, ValueError) as exc:
        if isinstance(exc, (InputError, ConfigurationError)):
            raise
        raise InputError(f"malformed problem description: {exc}") from exc


def save(inst: ProblemInstance, path: str):
    import json
    with open(path, "w") as fh:
        json.dump(to_json_dict(inst), fh)


def load(path: str, validate: bool = True) -> ProblemInstance:
    """Read a problem written by the reference's ``rapdb.problem.save``."""
    import json
    with open(path) as fh:
        return from_json_dict(json.load(fh), validate=validate)


def save_stack(inst: ProblemInstance, path: str):
    """Binary form for multi-GB instances (the JSON is impractical at C1/C2
    sizes): one .npz with the (m+1, n, n) stack and the vectors."""
    np.savez(path, n=inst.n, m=inst.m, p=inst.p, Q=inst.Q, q=inst.q, r=inst.r, A=inst.A, b=inst.b,
             lower=inst.primal_set.lower, upper=inst.primal_set.upper, mu=inst.mu, name=inst.name)


def load_stack(path: str, validate: bool = False) -> ProblemInstance:
    z = np.load(path, allow_pickle=False)
    return ProblemInstance(n=int(z["n"]), m=int(z["m"]), p=int(z["p"]), Q=z["Q"], q=z["q"], r=z["r"],
                           A=z["A"], b=z["b"], primal_set=Box(z["lower"], z["upper"]),
                           cone=NonnegOrthant(int(z["m"])), mu=float(z["mu"]), name=str(z["name"]),
                           validate=validate)
