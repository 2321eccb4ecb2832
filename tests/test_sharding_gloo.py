"""Multi-process check of the constraint-sharding decomposition (CPU, gloo).

Each of 2-3 ranks holds a contiguous block of the m+1 matrices (sharding.plan)
and runs the APDB-yx trial with exactly the exchange protocol of the device
path (include/rapdb_b200.h, rapdb_set_exchange): the partial
sum_i w_i (Q_i x_k + q_i) over local matrices is all-reduced (kind 1), local
g_i(x_new) are all-reduced as a zero-padded (m+1)-vector (kind 2), everything
else is replicated.  The accepted step sizes must equal the unsharded CPU
oracle's and the ranks must agree bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.sharding import ordered_allreduce_host, plan


def test_plan_balanced_and_contiguous():
    for m, R in [(10, 2), (10, 4), (200, 8), (512, 8), (5, 6), (3, 3)]:
        rngs = plan(m, R)
        assert rngs[0][0] == 0 and rngs[-1][1] == m + 1
        assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
        sizes = [k1 - k0 for k0, k1 in rngs]
        assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
    # an all-zero Q0 (C4) costs ~nothing: rank 0 takes one more matrix
    rngs = plan(5, 2, zero_flags=[True] + [False] * 5)
    assert rngs == [(0, 3), (3, 6)] or rngs[0][1] - rngs[0][0] >= rngs[1][1] - rngs[1][0]
    with pytest.raises(ValueError):
        plan(2, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_run(arr, k0, k1, allreduce, iters, nm):
    """APDB-yx with the device path's exchange protocol; returns (taus, x)."""
    n, m = arr.n, arr.m
    Q = arr.Q
    q = arr.q
    r = arr.r
    lo, hi = arr.lower, arr.upper

    def local_U(x):
        return {i: Q[i] @ x for i in range(k0, k1)}

    def g_full(U, x):
        loc = np.zeros(m + 1)
        for i, u in U.items():
            loc[i] = 0.5 * float(x @ u) + float(q[i] @ x) + r[i]
        return allreduce(loc)                       # exchange kind 2

    def grad(U, lam):
        part = np.zeros(n)
        for i, u in U.items():
            w = 1.0 if i == 0 else lam[i - 1]
            if w != 0.0:
                part = part + w * (u + q[i])
        return allreduce(part)                      # exchange kind 1 (no A block here)

    c_alpha, delta, eta = 0.4, 0.5, 0.7
    x = np.clip(np.zeros(n), lo, hi)
    lam = np.zeros(m)
    U = local_U(x)
    G = g_full(U, x)
    gy_cur = G[1:].copy()
    gy_prev = gy_cur.copy()
    tau_cand = tau_prev = 1.0
    gamma = 1.0
    sigma_prev = gamma * tau_cand
    alpha = c_alpha / sigma_prev
    phi_k = G[0] + float(lam @ G[1:])
    taus = []
    c_nm = 1.0 if nm else 0.0
    for _ in range(iters):
        tau = tau_cand
        slack = 1e-13 * (1.0 + abs(phi_k))
        while True:
            sigma = gamma * tau
            theta = sigma_prev / sigma
            lam_n = np.maximum(lam + sigma * ((1.0 + theta) * gy_cur - theta * gy_prev), 0.0)
            gx = grad(U, lam_n)
            x_n = np.clip(x - tau * gx, lo, hi)
            U_n = local_U(x_n)
            G_n = g_full(U_n, x_n)
            Dp = 0.5 * float((x_n - x) @ (x_n - x))
            Dd = 0.5 * float((lam_n - lam) @ (lam_n - lam))
            phi_new = G_n[0] + float(lam_n @ G_n[1:])
            phi_mix = G[0] + float(lam_n @ G[1:])
            lin = (phi_new - phi_mix) - float(gx @ (x_n - x))
            nrm = np.linalg.norm(G_n[1:] - gy_cur)
            alpha_n = c_alpha / sigma
            E = ((lin - Dp / tau) + nrm * nrm / (2.0 * alpha_n)) - (1.0 / sigma - theta * alpha) * Dd
            if E <= -(delta / tau) * Dp - (delta / sigma) * Dd + slack:
                break
            tau *= eta
        g_next = gamma * (1.0 + 0.0 * tau)
        tau_next = tau * np.sqrt((gamma / g_next) * (1.0 + c_nm * tau / tau_prev))
        gy_prev, gy_cur = gy_cur, G_n[1:].copy()
        x, lam, U, G = x_n, lam_n, U_n, G_n
        alpha, tau_prev, tau_cand, sigma_prev, gamma = alpha_n, tau, tau_next, sigma, g_next
        phi_k = phi_new
        taus.append(tau)
    return np.array(taus), x


def _worker(rank, world, port, iters, nm, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        arr = instances.dense_qcqp(40, 6, 5, seed=9)
        k0, k1 = plan(arr.m, world)[rank]

        def allreduce(v):     # the product's rank-ordered exchange (sharding.py)
            t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64).copy())
            ordered_allreduce_host([t])
            return t.numpy().copy()

        taus, x = _sharded_run(arr, k0, k1, allreduce, iters, nm)
        np.save(os.path.join(out, f"rank{rank}_taus.npy"), taus)
        np.save(os.path.join(out, f"rank{rank}_x.npy"), x)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nm", [(2, True), (3, False)])
def test_sharded_decomposition_gloo(tmp_path, world, nm):
    from oracle import rapdb_oracle as O
    iters = 120
    mp.spawn(_worker, args=(world, _free_port(), iters, nm, str(tmp_path)), nprocs=world, join=True)
    arr = instances.dense_qcqp(40, 6, 5, seed=9)
    eng = O.Engine(O.Problem.from_arrays(arr), O.Options(mode="yx", nonmonotone=nm), *O.initial_point(
        O.Problem.from_arrays(arr)))
    for _ in range(iters):
        eng.step()
    ref_taus = np.array([t.tau for t in eng.trace])
    xs = [np.load(tmp_path / f"rank{r}_x.npy") for r in range(world)]
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"rank{r}_taus.npy"), ref_taus)
        np.testing.assert_array_equal(xs[r], xs[0])            # replicas agree bit for bit
    assert np.linalg.norm(xs[0] - eng.x) <= 1e-12 * np.linalg.norm(eng.x)


def _ordered_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # contributions whose sum depends on the association: rank-ordered
        # ((p0 + p1) + p2) gives 1e16 in slot 0 (1e16 + 1 rounds back to
        # 1e16 twice), p0 + (p1 + p2) gives 1e16 + 2
        vals = {0: [1e16, 0.1, 3.0], 1: [1.0, 0.2, -1.0], 2: [1.0, 0.3, 2.0 ** -60]}[rank]
        t = torch.tensor(vals, dtype=torch.float64)
        t2 = torch.full((5,), float(rank + 1), dtype=torch.float64)
        ordered_allreduce_host([t, t2])
        np.save(os.path.join(out, f"ord{rank}.npy"), np.concatenate([t.numpy(), t2.numpy()]))
    finally:
        dist.destroy_process_group()


def test_ordered_allreduce_host_is_rank_ordered(tmp_path):
    """sharding.ordered_allreduce_host (the exchange of group_shard, and the
    association csrc/comm.cuh's NCCL exchange uses): every rank gets the same
    bits, equal to the left-to-right sum in rank order."""
    world = 3
    mp.spawn(_ordered_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = [np.load(tmp_path / f"ord{r}.npy") for r in range(world)]
    p = [np.array(v) for v in ([1e16, 0.1, 3.0], [1.0, 0.2, -1.0], [1.0, 0.3, 2.0 ** -60])]
    want = (p[0] + p[1]) + p[2]
    assert want[0] == 1e16 and (p[0] + (p[1] + p[2]))[0] == 1e16 + 2
    for g in got:
        np.testing.assert_array_equal(g[:3], want)
        np.testing.assert_array_equal(g[3:], np.full(5, 6.0))
        np.testing.assert_array_equal(g, got[0])
