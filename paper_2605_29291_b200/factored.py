"""Factored sparse QCQP instances (BASELINE config 3) on the device.

The reference can only hold such a problem as m+1 explicit operators
(``ProblemInstance`` problem.py:109-162; ``_as_operator`` :31-40 keeps sparse
ones as CSR) -- at n = 10^6 the products R_i^T R_i are not representable, so
config 3 is new capability built on the same operator contract
(problem.py:166-223, SURVEY.md section 8 row "C3"):

    Q_i = R_i^T R_i  (i = 0..mq, 0 = objective)   g_i = 1/2 |R_i x|^2 + c_i.x + d_i
    a_j x <= b_j     (j = 1..L)                    g_{mq+j} = a_j x - b_j   (Q = 0)

``FactoredInstance`` exposes the same surface the solver layers use from
``problem.ProblemInstance`` (n, m, p, primal_set, cone, mu, f/g evaluation,
device upload), so ``ApdbEngine`` / ``run_restarted`` / ``kkt_residual`` take
either.  HBM layout (``FactoredDeviceData``): every sparse operand as sliced
ELLPACK with slices of 32 slots (``SellMatrix`` / ``rapdb_sell``: a warp's
loads are coalesced with no staging, every row / column is summed in stored
order) -- the stacked R with its rows laid out per block in 128-row chunks,
A by row, and the transposes for the gradient gather (no atomics, fixed
summation order): R^T in ROW PHASES of at most ``RT_PHASE_ROWS`` stacked rows
(one Sell per phase over the columns sorted by entry count, each entry's row
tagged with its block id), so that each gather phase touches an L2-sized
slice of the W-cache and walking the phases walks every column in sorted row
order, and A^T the same way; plus the block id of every stacked row and
C [(mq+1) x n].
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .errors import ConfigurationError, InputError
from .geometry import Box, NonnegOrthant

import os as _os

# W-cache rows gathered per R^T phase (RAPDB_RT_PHASE_ROWS overrides; A/B
# runs): 2^22 rows = 32 MB of W, which stays resident in one half of the L2
RT_PHASE_ROWS = 1 << 22


def rt_phase_rows() -> int:
    return int(_os.environ.get("RAPDB_RT_PHASE_ROWS", str(RT_PHASE_ROWS)))


RT_MAX_PHASES = 8              # rapdb_set_factored_transpose
RT_TAG_SHIFT = 23              # tagged R^T rows: r | block << 23
W_CHUNK = 128                  # rows of W per |W_i|^2 partial (csrc/factored.cuh kWChunk)


class SellMatrix:
    """Sliced ELLPACK (slice height 32) of a CSR operand, host arrays.

    ``slot_rows[s]`` is the CSR row held by slot s (-1: padding); entry t of
    slot s is stored at ``sp[s // 32] + 32 t + s % 32`` and a slice is as wide
    as its longest slot.  Entries keep the CSR's stored order."""

    def __init__(self, M, slot_rows, idx_of=None, with_map=False):
        slot_rows = np.asarray(slot_rows, dtype=np.int64)
        nslots = slot_rows.size
        if nslots % 32:
            raise InputError("Sell needs a multiple of 32 slots")
        indptr = M.indptr.astype(np.int64)
        lens_rows = np.diff(indptr)
        valid = slot_rows >= 0
        ln = np.zeros(nslots, dtype=np.int32)
        ln[valid] = lens_rows[slot_rows[valid]]
        width = ln.reshape(-1, 32).max(axis=1).astype(np.int64) if nslots else np.zeros(0, np.int64)
        sp = np.zeros(nslots // 32 + 1, dtype=np.int64)
        np.cumsum(width * 32, out=sp[1:])
        tot = int(sp[-1])
        idx = np.zeros(tot, dtype=np.int32)
        val = np.zeros(tot, dtype=np.float64)
        if M.nnz:
            slot_of_row = np.full(M.shape[0], -1, dtype=np.int64)
            slot_of_row[slot_rows[valid]] = np.nonzero(valid)[0]
            row_of = np.repeat(np.arange(M.shape[0], dtype=np.int64), lens_rows)
            s = slot_of_row[row_of]
            if np.any(s < 0):
                raise InputError("Sell slots must cover every nonempty row")
            pos = sp[s >> 5] + (np.arange(M.nnz, dtype=np.int64) - indptr[row_of]) * 32 + (s & 31)
            ind = M.indices.astype(np.int64)
            idx[pos] = ind if idx_of is None else idx_of(ind)
            val[pos] = M.data
        self.nslots, self.sp, self.idx, self.val, self.len = nslots, sp, idx, val, ln
        self.map = slot_rows.astype(np.int32) if with_map else None
        self.entries = tot

    @classmethod
    def by_row(cls, M):
        """slot = row, padded to a multiple of 32."""
        nr = M.shape[0]
        slots = np.full(-(-nr // 32) * 32, -1, dtype=np.int64)
        slots[:nr] = np.arange(nr)
        return cls(M, slots)

    @classmethod
    def by_block_chunks(cls, M, rblk):
        """The stacked R: block i's rows start at slot 128 * (chunks of the
        earlier blocks), each block padded to whole 128-row chunks."""
        parts = []
        for i in range(len(rblk) - 1):
            r0, r1 = int(rblk[i]), int(rblk[i + 1])
            pad = -(-(r1 - r0) // W_CHUNK) * W_CHUNK
            part = np.full(pad, -1, dtype=np.int64)
            part[:r1 - r0] = np.arange(r0, r1)
            parts.append(part)
        return cls(M, np.concatenate(parts) if parts else np.zeros(0, np.int64))

    @classmethod
    def by_sorted_length(cls, M, idx_of=None):
        """Rows sorted by entry count (longest first, stable), so the slots
        of a slice have near-equal length; map = row of the slot."""
        nr = M.shape[0]
        order = np.argsort(-np.diff(M.indptr), kind="stable")
        slots = np.full(-(-nr // 32) * 32, -1, dtype=np.int64)
        slots[:nr] = order
        return cls(M, slots, idx_of=idx_of, with_map=True)


class DeviceSell:
    """A SellMatrix in HBM."""

    def __init__(self, m: SellMatrix, device):
        import torch

        def up(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            return torch.from_numpy(a if a.size else np.zeros(1, dtype=dt)).to(device)

        self.nslots, self.entries = m.nslots, m.entries
        self.sp, self.idx, self.val = up(m.sp, np.int64), up(m.idx, np.int32), up(m.val, np.float64)
        self.len = up(m.len, np.int32)
        self.map = None if m.map is None else up(m.map, np.int32)
        self._desc = None

    def descriptor(self):
        from ._capi import SellDescriptor
        if self._desc is None:
            self._desc = SellDescriptor(self.nslots, self.sp.data_ptr(), self.idx.data_ptr(), self.val.data_ptr(),
                                        self.len.data_ptr(), None if self.map is None else self.map.data_ptr())
        return self._desc


def phased_transpose(R, rmat, nph: int, tag: bool):
    """(bounds, [SellMatrix per phase]) of R^T split into nph row phases; rows
    tagged with their block id when ``tag``."""
    nr, n = R.shape
    bounds = np.array([nr * p // nph for p in range(nph + 1)], dtype=np.int64)
    mats = []
    for p in range(nph):
        Rt = R[bounds[p]:bounds[p + 1]].T.tocsr()      # sorted rows per column
        Rt.sort_indices()
        off = int(bounds[p])

        def idx_of(ind, off=off):
            ind = ind + off
            return ind | (rmat[ind].astype(np.int64) << RT_TAG_SHIFT) if tag else ind

        mats.append(SellMatrix.by_sorted_length(Rt, idx_of=idx_of))
    return bounds, mats


class FactoredInstance:
    """Q_i = R_i^T R_i QCQP with a sparse linear inequality block; box primal
    set, nonnegative-orthant cone over the m = mq + L constraints, p = 0."""

    def __init__(self, n, mq, R, rblk, C, d, A, b, lower, upper, mu=0.0, name=""):
        import scipy.sparse as sp
        self.n, self.mq = int(n), int(mq)
        self.R = sp.csr_matrix(R)
        self.rblk = np.asarray(rblk, dtype=np.int64)
        self.C = np.ascontiguousarray(C, dtype=np.float64)
        self.d = np.asarray(d, dtype=np.float64)
        self.A = sp.csr_matrix(A) if A is not None else sp.csr_matrix((0, self.n))
        self.b = np.asarray(b, dtype=np.float64).reshape(-1)
        self.L = self.A.shape[0]
        self.m = self.mq + self.L
        self.p = 0
        self.mu = float(mu)
        self.name = name
        self.dual_set = None
        self.primal_set = Box(np.asarray(lower, dtype=float), np.asarray(upper, dtype=float))
        self.cone = NonnegOrthant(self.m)
        n = self.n
        if n <= 0 or self.mq < 0:
            raise InputError("need n > 0 and mq >= 0")
        if self.R.shape[1] != n or self.A.shape[1] != n:
            raise InputError("R and A need n columns")
        if self.rblk.shape != (self.mq + 2,) or self.rblk[0] != 0 or self.rblk[-1] != self.R.shape[0] \
                or np.any(np.diff(self.rblk) < 0):
            raise InputError("rblk must be nondecreasing offsets 0..nr of the mq+1 blocks of R")
        if self.C.shape != (self.mq + 1, n) or self.d.shape != (self.mq + 1,):
            raise InputError("need C [(mq+1) x n] and d [mq+1]")
        if self.b.shape != (self.L,):
            raise InputError("b must have one entry per row of A")
        if self.primal_set.lower.shape != (n,) or self.primal_set.upper.shape != (n,):
            raise InputError("primal set dimension mismatch")
        if self.mu < 0:
            raise InputError("strong convexity modulus must be nonnegative")
        if self.R.shape[0] >= 2 ** 31 or self.R.nnz >= 2 ** 62:
            raise InputError("R too large for int32 row ids")
        self._dev = {}

    @classmethod
    def from_arrays(cls, arr, mu=0.0):
        """From ``instances.FactoredArrays``."""
        rblk = np.arange(arr.mq + 2, dtype=np.int64) * arr.rows
        return cls(arr.n, arr.mq, arr.R, rblk, arr.C, arr.d, arr.A, arr.b, arr.lower, arr.upper,
                   mu=mu, name=arr.name)

    def check_device_support(self):
        return None

    # -- device ---------------------------------------------------------------
    def shard_ranges(self, nranks: int):
        """Constraint shards: contiguous quadratic
        blocks balanced by R rows (block 0 = objective counts like any other)
        and an even split of the linear rows; [(k0, k1, l0, l1)] per rank."""
        nb = self.mq + 1
        if nranks < 1 or nranks > nb:
            raise ConfigurationError(f"cannot shard {nb} quadratic blocks over {nranks} ranks")
        rows = np.diff(self.rblk).astype(float) + 1.0
        cum = np.concatenate([[0.0], np.cumsum(rows)])
        bounds = [0]
        for r in range(1, nranks):
            k = int(np.searchsorted(cum, cum[-1] * r / nranks, side="left"))
            k = min(max(k, bounds[-1] + 1), nb - (nranks - r))
            bounds.append(k)
        bounds.append(nb)
        return [(bounds[r], bounds[r + 1], self.L * r // nranks, self.L * (r + 1) // nranks)
                for r in range(nranks)]

    def device_data(self, device=None, pinned_host=None, krange=None, lrange=None):
        """Upload (cached per device and shard).  krange = (k0, k1): quadratic
        blocks held by this rank, lrange = (l0, l1): its linear rows."""
        import torch
        k0, k1 = krange if krange is not None else (0, self.mq + 1)
        l0, l1 = lrange if lrange is not None else (0, self.L)
        if krange is not None and lrange is None and tuple(krange) != (0, self.mq + 1):
            raise ConfigurationError("a factored shard needs both its block range and its linear-row range")
        dev = torch.device("cuda", 0) if device is None else torch.device(device)
        key = str(dev) if (k0, k1, l0, l1) == (0, self.mq + 1, 0, self.L) else f"{dev}[{k0}:{k1}|{l0}:{l1}]"
        key += f"/ph{rt_phase_rows()}"
        if key not in self._dev:
            self._dev[key] = FactoredDeviceData.upload(self, dev, k0, k1, l0, l1)
        return self._dev[key]

    def drop_device_data(self):
        for k in [k for k in self._dev if not k.startswith("_")]:
            del self._dev[k]

    # -- evaluations (problem.py:166-186) on the device ----------------------
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
        return np.zeros(0)

    def project_dual_cone(self, lam):
        return np.maximum(np.asarray(lam, dtype=float), 0.0)


class SparseQInstance(FactoredInstance):
    """A QCQP whose quadratic forms are sparse symmetric matrices, kept sparse.

    The reference stores a ``Q_i`` with fewer than 25 % nonzeros as CSR
    (``_as_operator`` problem.py:31-40) and applies it with scipy's
    ``csr_matvec``; ``problem.ProblemInstance`` here densifies every ``Q_i``
    for the packed dense sweep, which a large sparse stack does not survive.
    This instance keeps the stack sparse on the device: the stacked
    ``Q_0..Q_m`` ride the factored path's row pass as one Sell operand with n
    rows per block (``rapdb_set_factored_symmetric``) -- ``u_i = Q_i x`` summed
    in CSR order (the bits of the reference's products), ``g_i = 1/2 x.u_i +
    q_i.x + r_i``, ``grad_x Phi = sum_i w_i (u_i + q_i) + A^T mu`` in the
    reference's operation order (problem.py:205-214), no transposed gather.
    Constraints: ``m`` quadratic rows plus optional sparse linear rows
    ``A x <= b`` (orthant cone), box primal set, no equality block, no
    adaptive restart (as for every factored instance)."""

    sym = True

    def __init__(self, n, m, Q, q, r, lower, upper, A=None, b=None, mu=0.0, name="", symmetry_tol=1e-12):
        import scipy.sparse as sp
        n, m = int(n), int(m)
        if len(Q) != m + 1:
            raise InputError("need m+1 quadratic forms (objective plus m constraints)")
        mats = []
        for i, M in enumerate(Q):
            M = sp.csr_matrix(M)
            if M.shape != (n, n):
                raise InputError(f"quadratic form {i} has wrong dimensions")
            d = abs(M - M.T)
            if d.nnz and d.max() > symmetry_tol * max(1.0, abs(M).max()):
                raise InputError(f"quadratic form {i} is not symmetric")
            mats.append(M)
        R = sp.vstack(mats, format="csr") if mats else sp.csr_matrix((0, n))
        rblk = np.arange(m + 2, dtype=np.int64) * n
        q = np.asarray(q, dtype=np.float64).reshape(m + 1, n)
        L = 0 if A is None else sp.csr_matrix(A).shape[0]
        super().__init__(n, m, R, rblk, q, np.asarray(r, dtype=np.float64), A,
                         np.zeros(0) if b is None else b, lower, upper, mu=mu, name=name)
        assert self.L == L

    @classmethod
    def from_problem(cls, inst, density_limit: float = 0.25):
        """From a ``problem.ProblemInstance`` (box primal set, orthant cone, p = 0)
        whose forms are all below the reference's CSR density limit."""
        import scipy.sparse as sp
        if inst.p != 0:
            raise ConfigurationError("a sparse-Q instance has no equality block")
        if not isinstance(inst.primal_set, Box) or not isinstance(inst.cone, NonnegOrthant):
            raise ConfigurationError("a sparse-Q instance needs a box primal set and the orthant cone")
        Q = [sp.csr_matrix(inst.Q[i]) for i in range(inst.m + 1)]
        for i, M in enumerate(Q):
            if M.nnz > density_limit * inst.n * inst.n:
                raise ConfigurationError(f"quadratic form {i} is not sparse (the reference would keep it dense)")
        return cls(inst.n, inst.m, Q, inst.q, inst.r, inst.primal_set.lower, inst.primal_set.upper,
                   mu=inst.mu, name=getattr(inst, "name", ""))


class FactoredDeviceData:
    """A FactoredInstance resident in HBM (see module docstring)."""

    factored = True

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @classmethod
    def upload(cls, inst: FactoredInstance, device, k0=0, k1=None, l0=0, l1=None):
        import torch
        k1 = inst.mq + 1 if k1 is None else k1
        l1 = inst.L if l1 is None else l1

        def f64(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)

        def i64(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(device)

        def i32(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)

        r0, r1 = int(inst.rblk[k0]), int(inst.rblk[k1])
        R = inst.R[r0:r1]              # stored entry order kept: it is the summation order of W = R x
        rblk = inst.rblk[k0:k1 + 1] - r0
        A = inst.A[l0:l1]
        At = A.T.tocsr()
        At.sort_indices()              # a column's entries in row order
        nr = R.shape[0]
        rmat = np.repeat(np.arange(k1 - k0, dtype=np.int32), np.diff(rblk))
        sym = bool(getattr(inst, "sym", False))
        if sym:     # the blocks are the Q_i themselves: nothing to gather through R^T
            import scipy.sparse as sp
            nph, tag = 1, False
            rt_bounds = np.array([0, nr], dtype=np.int64)
            rt_mats = [SellMatrix.by_sorted_length(sp.csr_matrix((inst.n, nr)))]
        else:
            nph = min(RT_MAX_PHASES, max(1, -(-nr // rt_phase_rows())))
            tag = nr <= (1 << RT_TAG_SHIFT) and (k1 - k0) <= 256
            rt_bounds, rt_mats = phased_transpose(R, rmat, nph, tag)
        sell_R = SellMatrix.by_block_chunks(R, rblk)
        sell_A = SellMatrix.by_row(A)
        sell_AT = SellMatrix.by_sorted_length(At)
        one = lambda t: t if t.numel() else torch.zeros(1, dtype=t.dtype, device=device)
        return cls(n=inst.n, m=inst.m, p=0, mq=inst.mq, L=inst.L, nr=nr, rblk=rblk.copy(),
                   k0=k0, k1=k1, l0=l0, l1=l1,
                   sell_R=DeviceSell(sell_R, device), sell_A=DeviceSell(sell_A, device),
                   sell_RT=[DeviceSell(t, device) for t in rt_mats], sell_AT=DeviceSell(sell_AT, device),
                   rmat=one(i32(rmat)), C=one(f64(inst.C[k0:k1])), d=one(f64(inst.d[k0:k1])),
                   b=one(f64(inst.b[l0:l1])), lower=f64(inst.primal_set.lower),
                   upper=f64(inst.primal_set.upper), mu=inst.mu, device=device,
                   nnz_r=int(R.nnz), nnz_a=int(A.nnz), rt_nph=nph, rt_bounds=rt_bounds, rt_tag=int(tag), sym=sym)
