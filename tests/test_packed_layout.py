"""The packed symmetric Q-stack layout (csrc/symsweep.cuh): geometry on the
host (no GPU), pack / sweep / solve parity on the device.

Layout: 32 x 32 row-major sub-tiles in 64 x 64 units, units block-row-major
over Bi <= Bj, a diagonal unit storing sub-tiles (0,0), (0,1), (1,1); ragged
edges zero padded.  The Python mirror below reconstructs the dense matrix from
the packed buffer so the device pack can be checked element for element."""

import ctypes
import os

import numpy as np
import pytest

from conftest import REPO
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.problem import packed_source_elements

LIB = os.path.join(REPO, "paper_2605_29291_b200", "_rapdb_b200.so")


def units_of(n):
    """[(bi, bj, [(sr, sc), ...])] in storage order (symsweep.cuh fill_units)."""
    nb32 = (n + 31) // 32
    nbB = (nb32 + 1) // 2
    out = []
    for bi in range(nbB):
        rs = 2 if 2 * bi + 1 < nb32 else 1
        for bj in range(bi, nbB):
            cs = 2 if 2 * bj + 1 < nb32 else 1
            if bi == bj:
                subs = [(0, 0)] + ([(0, 1), (1, 1)] if rs == 2 else [])
            else:
                subs = [(a, b) for a in range(rs) for b in range(cs)]
            out.append((bi, bj, subs))
    return out


def packed_len(n):
    return sum(len(s) for _, _, s in units_of(n)) * 1024


def unpack(buf, n):
    """Dense symmetric n x n matrix from one packed matrix (host mirror)."""
    nb = ((n + 31) // 32) * 32
    D = np.zeros((nb + 32, nb + 32))
    k = 0
    for bi, bj, subs in units_of(n):
        for sr, sc in subs:
            r0, c0 = (2 * bi + sr) * 32, (2 * bj + sc) * 32
            T = buf[k * 1024:(k + 1) * 1024].reshape(32, 32)
            D[r0:r0 + 32, c0:c0 + 32] = T
            if r0 != c0:
                D[c0:c0 + 32, r0:r0 + 32] = T.T
            k += 1
    return D[:n, :n]


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 64, 65, 96, 127, 128, 200, 1001, 2000, 4096])
def test_packed_size_matches_library(n):
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    lib = ctypes.CDLL(LIB)
    lib.rapdb_packed_doubles.argtypes = [ctypes.c_int]
    lib.rapdb_packed_doubles.restype = ctypes.c_longlong
    assert lib.rapdb_packed_doubles(n) == packed_len(n)


@pytest.mark.parametrize("n", [1, 31, 33, 64, 65, 200, 2000])
def test_packed_source_elements(n):
    # entries of the upper 32-block triangle incl. the diagonal blocks
    nb32 = (n + 31) // 32
    ext = [min(32, n - 32 * k) for k in range(nb32)]
    full = sum(e * e for e in ext) + sum(ext[i] * ext[j] for i in range(nb32) for j in range(i + 1, nb32))
    assert packed_source_elements(n) == full
    assert n * (n + 1) // 2 <= packed_source_elements(n) <= n * n


def test_packed_halves_the_stack():
    for n in (2000, 4096):
        assert packed_len(n) / (n * n) < 0.53


# ------------------------------------------------------------------ device

def _sym(rng, k, n):
    M = rng.standard_normal((k, n, n))
    return np.ascontiguousarray(0.5 * (M + M.transpose(0, 2, 1)))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 33, 64, 65, 130, 257])
@pytest.mark.parametrize("src", ["device", "pinned"])
def test_pack_kernel_exact(n, src):
    import torch
    from paper_2605_29291_b200 import _capi
    rng = np.random.default_rng(n)
    Q = _sym(rng, 3, n)
    t = torch.from_numpy(Q)
    t = t.cuda() if src == "device" else t.pin_memory()
    spm = _capi.packed_doubles(n)
    out = torch.full((3, spm), np.nan, dtype=torch.float64, device="cuda")
    _capi.pack_symmetric(n, 3, t.data_ptr(), n, n * n, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    host = out.cpu().numpy()
    assert not np.isnan(host).any()
    for i in range(3):
        np.testing.assert_array_equal(unpack(host[i], n), Q[i])


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(1, 1), (33, 2), (65, 3), (200, 10), (257, 5), (1001, 7)])
def test_packed_sweep_matches_numpy(n, m, monkeypatch):
    import torch
    monkeypatch.setenv("RAPDB_LAYOUT", "packed")
    arr = instances.dense_qcqp(n, m, max(1, min(9, n)), seed=5)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    ev = inst._evaluator()
    assert ev.data.layout == "packed"
    x = np.random.default_rng(2).uniform(-1, 1, n)
    u, g, _ = ev.ctx.probe_sweep(torch.from_numpy(x).cuda(), reps=3)
    u = u.cpu().numpy()
    for i in range(m + 1):
        ref = arr.Q[i] @ x
        assert np.max(np.abs(u[i] - ref)) <= 1e-13 * (1 + np.max(np.abs(ref)))
    gref = np.array([0.5 * x @ (arr.Q[i] @ x) + arr.q[i] @ x + arr.r[i] for i in range(m + 1)])
    np.testing.assert_allclose(g.cpu().numpy(), gref, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_packed_and_rows_layouts_agree(monkeypatch):
    """Same instance through both layouts: identical accepted step sizes,
    iterates within 1e-11 (the sums run in different orders)."""
    arr = instances.dense_qcqp(300, 12, 15, seed=8)
    out = {}
    for layout in ("rows", "packed"):
        monkeypatch.setenv("RAPDB_LAYOUT", layout)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
        res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(60), budget=200)
        out[layout] = res
    a, b = out["rows"], out["packed"]
    ta = np.array([[t.tau_start, t.tau, t.evals_iter] for t in a.trace])
    tb = np.array([[t.tau_start, t.tau, t.evals_iter] for t in b.trace])
    np.testing.assert_array_equal(ta, tb)
    assert np.linalg.norm(a.solution.x - b.solution.x) <= 1e-11 * (1 + np.linalg.norm(a.solution.x))


@pytest.mark.gpu
def test_device_generated_instance_vs_oracle():
    """DeviceDenseInstance (stack generated and packed on the GPU): unpack the
    stack, run the CPU oracle on it, compare the first 100 accepted steps."""
    import torch
    from oracle import rapdb_oracle as O
    from paper_2605_29291_b200 import _capi
    n, m = 97, 6
    inst = R.DeviceDenseInstance(n, m, 8, seed=3)
    data = inst.device_data(torch.device("cuda", 0))
    host = data.Q.cpu().numpy()
    Q = np.stack([unpack(host[i], n) for i in range(m + 1)])
    np.testing.assert_array_equal(Q, np.transpose(Q, (0, 2, 1)))
    assert np.linalg.eigvalsh(Q[1])[0] >= 0.1 - 1e-9
    arr = instances.QcqpArrays(n=n, m=m, p=0, Q=Q, q=inst.q, r=inst.r, A=np.zeros((0, n)), b=np.zeros(0),
                               lower=inst.primal_set.lower, upper=inst.primal_set.upper)
    ref = O.run_restarted(O.Problem.from_arrays(arr), O.Options(mode="yx", nonmonotone=False),
                          O.Policy("fixed", period=50), budget=100)
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.FixedRestart(50), budget=100)
    a = np.array([[t.tau_start, t.tau, t.evals_iter] for t in res.trace])
    b = np.array([[t.tau_start, t.tau, t.evals_iter] for t in ref.trace])
    np.testing.assert_array_equal(a, b)
    assert np.linalg.norm(res.solution.x - ref.x) <= 1e-9 * (1 + np.linalg.norm(ref.x))


@pytest.mark.gpu
def test_nearly_symmetric_input_uses_upper_triangle(monkeypatch):
    """A stack symmetric only to ~1e-13 (inside the reference's 1e-12
    validation tolerance): the packed operator is the upper triangle, so u
    differs from the row-major product by at most the asymmetry applied to |x|."""
    import torch
    arr = instances.dense_qcqp(150, 4, 10, seed=9)
    rng = np.random.default_rng(0)
    Q = arr.Q + 1e-13 * rng.standard_normal(arr.Q.shape)
    arr.Q = np.ascontiguousarray(Q)
    x = rng.uniform(-1, 1, 150)
    us = {}
    for layout in ("rows", "packed"):
        monkeypatch.setenv("RAPDB_LAYOUT", layout)
        inst = R.ProblemInstance.from_arrays(arr, validate=True)
        u, _, _ = inst._evaluator().ctx.probe_sweep(torch.from_numpy(x).cuda())
        us[layout] = u.cpu().numpy()
    # |u_rows - u_packed|_i <= sum_j |Q_ij - Q_ji| |x_j| (+ rounding)
    asym = np.abs(arr.Q - np.transpose(arr.Q, (0, 2, 1))) @ np.abs(x)
    assert np.all(np.abs(us["rows"] - us["packed"]) <= asym + 1e-13 * (1 + np.max(np.abs(us["rows"]))))
    assert np.max(asym) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,p", [(1, 1, 0), (33, 2, 0), (65, 3, 1), (130, 4, 2), (257, 1, 0)])
def test_packed_solver_ragged_vs_oracle(n, m, p, monkeypatch):
    """Whole solves on ragged n (edge units with one sub-row / column, padded
    sub-tiles) with equality rows: accepted steps identical to the oracle."""
    from oracle import rapdb_oracle as O
    monkeypatch.setenv("RAPDB_LAYOUT", "packed")
    arr = instances.dense_qcqp(n, m, max(1, min(6, n)), seed=11 + n)
    if p:
        rng = np.random.default_rng(n)
        arr.A = rng.standard_normal((p, n))
        arr.b = arr.A @ rng.uniform(-0.1, 0.1, n)
        arr.p = p
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    P = O.Problem.from_arrays(arr)
    for nm in (False, True):
        ref = O.run_restarted(P, O.Options(mode="yx", nonmonotone=nm), O.Policy("fixed", period=40), budget=100)
        res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.FixedRestart(40), budget=100)
        a = np.array([[t.tau_start, t.tau, t.evals_iter] for t in res.trace])
        b = np.array([[t.tau_start, t.tau, t.evals_iter] for t in ref.trace])
        np.testing.assert_array_equal(a, b)
        assert np.linalg.norm(res.solution.x - ref.x) <= 1e-9 * (1 + np.linalg.norm(ref.x))


@pytest.mark.gpu
def test_xglobal_mode_is_bitwise_identical(monkeypatch):
    """Long-x fallback (each consumer warp loads its unit's two x blocks
    instead of staging all of x in shared memory), forced at a small n: the
    same arithmetic on the same values -> bit-identical solves."""
    arr = instances.dense_qcqp(333, 6, 9, seed=12)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("RAPDB_XGLOBAL", flag)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
        out[flag] = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(50),
                                    budget=150)
    a, b = out["0"], out["1"]
    np.testing.assert_array_equal(np.array([[t.tau, t.evals_iter] for t in a.trace]),
                                  np.array([[t.tau, t.evals_iter] for t in b.trace]))
    np.testing.assert_array_equal(a.solution.x, b.solution.x)


@pytest.mark.gpu
@pytest.mark.slow
def test_long_x_instance_vs_oracle():
    """n = 20 500 (x no longer fits in shared memory next to the ring: the
    automatic long-x path), first 4 iterations against the oracle."""
    from oracle import rapdb_oracle as O
    arr = instances.dense_qcqp(20_500, 1, 3, seed=2)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    P = O.Problem.from_arrays(arr)
    eng = O.Engine(P, O.Options(mode="yx", nonmonotone=False), *O.initial_point(P))
    for _ in range(4):
        eng.step()
    dev = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.initial_iterate(inst))
    dev.run_block(4)
    np.testing.assert_array_equal(np.array([[t.tau_start, t.tau, t.evals_iter] for t in dev.trace]),
                                  np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace]))
    assert np.linalg.norm(dev.last.x - eng.x) <= 1e-9 * (1 + np.linalg.norm(eng.x))


@pytest.mark.gpu
@pytest.mark.parametrize("n,m", [(97, 23), (333, 40), (1001, 17)])
def test_early_reduction_is_bitwise_identical(n, m, monkeypatch):
    """Unit partials reduced by the slot-less warp during the stream (matrix
    chunks) or all after it: the same K-order sums whichever warp runs an
    item, so the sweep outputs and whole solves are bit-identical for any
    chunk count (ragged n; 2, 3, 7 and 64 chunks; with the long-x path)."""
    import torch
    arr = instances.dense_qcqp(n, m, max(1, min(9, n)), seed=21)
    x = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, n)).cuda()
    ref = None
    for chunks, xg in (("0", "0"), ("2", "0"), ("3", "0"), ("7", "0"), ("64", "0"), ("5", "1")):
        monkeypatch.setenv("RAPDB_EARLY_CHUNKS", chunks)
        monkeypatch.setenv("RAPDB_XGLOBAL", xg)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
        ev = inst._evaluator()
        u, g, _ = ev.ctx.probe_sweep(x, reps=4)
        res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(40), budget=120)
        got = (u.cpu().numpy(), g.cpu().numpy(), np.array([[t.tau, t.evals_iter] for t in res.trace]),
               res.solution.x)
        if ref is None:
            ref = got
            uref = np.stack([arr.Q[i] @ x.cpu().numpy() for i in range(m + 1)])
            assert np.max(np.abs(got[0] - uref)) <= 1e-13 * (1 + np.max(np.abs(uref)))
            continue
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)
