"""Constraint-sharded execution on one GPU.

* forced "split" mode with one rank stops at every exchange point and resumes in
  a new launch -- it must be bit-identical to the fused single-launch path;
* R emulated shards (one context per shard, host threads meeting at each
  exchange, rank-ordered sums) must reproduce the reference's accepted step
  sizes and iterates like the unsharded path.
The library's own NCCL communicator runs at world size 1 (one GPU per box),
and two real processes share the GPU with a gloo rank-ordered exchange
(bottom of this file); tests/test_sharding_gloo.py runs the exchange
(sharding.ordered_allreduce_host) over gloo on CPU at world size 2-3.
"""

import numpy as np
import pytest

from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.sharding import EmulatedCluster, Shard
from test_gpu_parity import TAU, crit, inst_from, rel, trace_arr

pytestmark = pytest.mark.gpu


def _solve(inst, shard=None, mode="yx", nm=True, policy=None, budget=300, eps=None):
    return R.run_restarted(inst, R.SolverConfig(mode=mode, nonmonotone=nm), policy or R.FixedRestart(40),
                           budget=budget, criteria=crit(eps), shard=shard)


@pytest.mark.parametrize("mode,policy", [("yx", "fixed"), ("xy", "fixed"), ("yx", "adaptive")])
def test_split_single_rank_is_bitwise_identical(mode, policy):
    arr = instances.dense_qcqp(150, 9, 12, seed=4)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    pol = R.FixedRestart(40) if policy == "fixed" else R.AdaptiveRestart(warmup=30, check_period=60)
    fused = _solve(inst, None, mode, True, pol, 300, 1e-9)
    calls = []
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True,
                  exchange=lambda views: calls.append(len(views)))
    split = _solve(inst, shard, mode, True, pol, 300, 1e-9)
    assert calls, "split mode never reached an exchange point"
    np.testing.assert_array_equal(trace_arr(split.trace)[:, :7], trace_arr(fused.trace)[:, :7])
    np.testing.assert_array_equal(split.solution.x, fused.solution.x)
    np.testing.assert_array_equal(split.solution.lam, fused.solution.lam)
    assert [e.iteration for e in split.restart_log] == [e.iteration for e in fused.restart_log]


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("key,mode,nm", [("yx_mono", "yx", False), ("yx_nm", "yx", True), ("xy_nm", "xy", True)])
def test_emulated_shards_small_qcqp(nranks, key, mode, nm):
    g = load_golden("small_qcqp")
    inst = inst_from(g["Q"], g["q"], g["r"], g["lower"], g["upper"])
    cluster = EmulatedCluster(nranks)

    def body(shard):
        eng = R.ApdbEngine(inst, R.SolverConfig(mode=mode, nonmonotone=nm), R.initial_iterate(inst), shard=shard)
        eng.run_block(200)
        return trace_arr(eng.trace), eng.last

    outs = cluster.run(inst, body)
    for tr, z in outs:
        np.testing.assert_array_equal(tr[:, TAU], g[f"{key}/trace"][:200, TAU])
        assert rel(z.x, g[f"{key}/snap_x"][-1]) <= 1e-9
        assert rel(z.lam, g[f"{key}/snap_lam"][-1]) <= 1e-9
    for tr, z in outs[1:]:      # replicas agree bit for bit
        np.testing.assert_array_equal(z.x, outs[0][1].x)


@pytest.mark.parametrize("nranks", [2, 4])
def test_emulated_shards_c0_restarts_and_kkt(nranks):
    g = load_golden("c0")
    arr = instances.config_instance("C0")
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    cluster = EmulatedCluster(nranks)

    def body(shard):
        return R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.NoRestart(),
                               budget=50000, criteria=crit(1e-6), shard=shard)

    for res in cluster.run(inst, body):
        tr = trace_arr(res.trace)
        np.testing.assert_array_equal(tr[:200, TAU], g["mono_none/trace"][:200, TAU])
        assert res.converged and res.iterations == int(g["mono_none/iterations"])
        assert abs(res.metrics.f_value - g["mono_none/metrics"][5]) <= 1e-9 * abs(g["mono_none/metrics"][5])


def test_emulated_shards_adaptive_gap():
    g = load_golden("small_qcqp")
    inst = inst_from(g["Q"], g["q"], g["r"], g["lower"], g["upper"])
    cluster = EmulatedCluster(2)

    def body(shard):
        return R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True),
                               R.AdaptiveRestart(warmup=50, check_period=100), budget=1500,
                               criteria=crit(1e-8), shard=shard)

    ref_it = list(g["yx_nm_ada/restart_iters"])
    ref_gaps = g["yx_nm_ada/restart_gaps"]
    meaningful = [it for it, (gn, gr) in zip(ref_it, ref_gaps) if gr > 1e-8]
    for res in cluster.run(inst, body):
        np.testing.assert_array_equal(trace_arr(res.trace)[:200, TAU], g["yx_nm_ada/trace"][:200, TAU])
        assert [e.iteration for e in res.restart_log][:len(meaningful)] == meaningful


@pytest.mark.parametrize("nranks", [2, 3])
def test_emulated_shards_kml_zero_objective_and_equality(nranks):
    """C4's structure (all-zero Q_0 never streamed, one equality row, a free
    epigraph variable) sharded: the zero matrix lands on rank 0's range."""
    g = load_golden("kml_small")
    arr = instances.kml_epigraph(N=120, d=10)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    cluster = EmulatedCluster(nranks)

    def body(shard):
        return R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(500),
                               budget=3000, criteria=crit(1e-6), shard=shard)

    for res in cluster.run(inst, body):
        tr = trace_arr(res.trace)
        np.testing.assert_array_equal(tr[:200, TAU], g["nm_fixed500/trace"][:200, TAU])
        assert res.iterations == int(g["nm_fixed500/iterations"])


def test_emulated_shards_factored_xy():
    """xy mode (two gradient exchanges per trial) on a sharded factored instance."""
    from conftest import FACTORED_SMALL
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(**FACTORED_SMALL)
    inst = FactoredInstance.from_arrays(arr)
    cfg = R.SolverConfig(mode="xy", nonmonotone=True)
    ref = R.ApdbEngine(inst, cfg, R.initial_iterate(inst))
    ref.run_block(60)
    cluster = EmulatedCluster(2)

    def body(shard):
        eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst), shard=shard)
        eng.run_block(60)
        return trace_arr(eng.trace), eng.last

    for tr, z in cluster.run(inst, body):
        np.testing.assert_array_equal(tr[:, 5], trace_arr(ref.trace)[:, 5])
        np.testing.assert_array_equal(tr[:, 1:5], trace_arr(ref.trace)[:, 1:5])
        assert rel(z.x, ref.last.x) <= 1e-11


@pytest.mark.parametrize("mode,policy", [("yx", "fixed"), ("xy", "fixed"), ("yx", "adaptive")])
def test_peer_exchange_single_rank_is_bitwise_identical(mode, policy):
    """The in-kernel NVLink exchange path (push to every peer's slot, release
    / acquire generation flags, rank-ordered sum) with one rank: it must leave
    every result bit-identical to the fused run (the sum of one slot).  The
    smoothed gap's H still goes through the host callback (adaptive case)."""
    arr = instances.dense_qcqp(150, 9, 12, seed=4)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    pol = R.FixedRestart(40) if policy == "fixed" else R.AdaptiveRestart(warmup=30, check_period=60)
    fused = _solve(inst, None, mode, True, pol, 300, 1e-9)
    calls = []
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True, p2p=True,
                  exchange=lambda views: calls.append(len(views)))
    peer = _solve(inst, shard, mode, True, pol, 300, 1e-9)
    if policy == "fixed":
        assert not calls, "gradient / g exchanges must not leave the kernel"
    np.testing.assert_array_equal(trace_arr(peer.trace)[:, :7], trace_arr(fused.trace)[:, :7])
    np.testing.assert_array_equal(peer.solution.x, fused.solution.x)
    np.testing.assert_array_equal(peer.solution.lam, fused.solution.lam)


# --------------------------------------------------------------------------
# The library's own NCCL communicator (csrc/comm.cuh) and real multi-process
# shards.  Only one GPU is available per test box: NCCL refuses two ranks on
# one device, so the native communicator runs at world size 1 here (split
# mode, every exchange through rapdb_comm: bitwise identity with the fused
# run), and the multi-process path runs its exchanges through a gloo group
# (sharding.group_shard) -- the kernels stop at each exchange point, so the
# processes never spin on each other on the shared GPU.


def _native_comm():
    from paper_2605_29291_b200 import _capi
    return _capi.Comm(0, _capi.comm_unique_id(), 0, 1)


@pytest.mark.parametrize("mode,policy", [("yx", "fixed"), ("xy", "fixed"), ("yx", "adaptive")])
def test_native_comm_single_rank_is_bitwise_identical(mode, policy):
    arr = instances.dense_qcqp(150, 9, 12, seed=4)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    pol = R.FixedRestart(40) if policy == "fixed" else R.AdaptiveRestart(warmup=30, check_period=60)
    fused = _solve(inst, None, mode, True, pol, 300, 1e-9)
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True, comm=_native_comm(), name="nccl")
    eng = R.ApdbEngine(inst, R.SolverConfig(mode=mode, nonmonotone=True), R.initial_iterate(inst), shard=shard)
    eng.run_block(5)
    assert eng._ctx.exchange_count() > 0, "split mode never reached the native exchange"
    split = _solve(inst, shard, mode, True, pol, 300, 1e-9)
    np.testing.assert_array_equal(trace_arr(split.trace)[:, :7], trace_arr(fused.trace)[:, :7])
    np.testing.assert_array_equal(split.solution.x, fused.solution.x)
    np.testing.assert_array_equal(split.solution.lam, fused.solution.lam)


def test_native_comm_factored_single_rank():
    from conftest import FACTORED_SMALL
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(**FACTORED_SMALL)
    inst = FactoredInstance.from_arrays(arr)
    cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    ref = R.ApdbEngine(inst, cfg, R.initial_iterate(inst))
    ref.run_block(60)
    k0, k1, l0, l1 = inst.shard_ranges(1)[0]
    shard = Shard(rank=0, nranks=1, k0=k0, k1=k1, l0=l0, l1=l1, force_split=True, comm=_native_comm())
    eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst), shard=shard)
    eng.run_block(60)
    np.testing.assert_array_equal(trace_arr(eng.trace)[:, :7], trace_arr(ref.trace)[:, :7])
    np.testing.assert_array_equal(eng.last.x, ref.last.x)


def test_native_comm_allreduce_world_one_is_identity():
    import torch
    comm = _native_comm()
    for n in (7, 3 << 20):        # the all-gather and the send/recv + all-gather paths
        t = torch.randn(n, dtype=torch.float64, device="cuda")
        before = t.clone()
        comm.allreduce_ordered(t, torch.cuda.current_stream().cuda_stream)
        assert torch.equal(t, before)


def _group_worker(rank, world, port, out, kind):
    import os
    import torch
    import torch.distributed as dist
    from paper_2605_29291_b200.sharding import group_shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        if kind == "dense":
            arr = instances.dense_qcqp(150, 9, 12, seed=4)
            inst = R.ProblemInstance.from_arrays(arr, validate=False)
            cfg = R.SolverConfig(mode="yx", nonmonotone=True)
            pol = R.FixedRestart(40)
        else:
            from conftest import FACTORED_SMALL
            from paper_2605_29291_b200.factored import FactoredInstance
            inst = FactoredInstance.from_arrays(instances.factored_qcqp(**FACTORED_SMALL))
            cfg = R.SolverConfig(mode="yx", nonmonotone=False)
            pol = R.FixedRestart(50)
        res = R.run_restarted(inst, cfg, pol, budget=150, criteria=crit(1e-9), shard=group_shard(inst))
        np.save(os.path.join(out, f"{kind}{rank}_trace.npy"), trace_arr(res.trace)[:, :7])
        np.save(os.path.join(out, f"{kind}{rank}_x.npy"), res.solution.x)
        np.save(os.path.join(out, f"{kind}{rank}_lam.npy"), res.solution.lam)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["dense", "factored"])
def test_two_processes_one_gpu_group_exchange(tmp_path, kind):
    """Two real processes, each binding its own constraint shard on the GPU and
    running run_restarted(shard=group_shard(...)) with a rank-ordered gloo
    exchange: both ranks agree bit for bit with each other and with the
    emulated 2-rank cluster (the same rank-ordered sums), and the accepted
    step sizes equal the unsharded run's."""
    import torch.multiprocessing as mp
    from test_sharding_gloo import _free_port
    world = 2
    mp.spawn(_group_worker, args=(world, _free_port(), str(tmp_path), kind), nprocs=world, join=True)
    if kind == "dense":
        arr = instances.dense_qcqp(150, 9, 12, seed=4)
        inst = R.ProblemInstance.from_arrays(arr, validate=False)
        cfg, pol = R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(40)
    else:
        from conftest import FACTORED_SMALL
        from paper_2605_29291_b200.factored import FactoredInstance
        inst = FactoredInstance.from_arrays(instances.factored_qcqp(**FACTORED_SMALL))
        cfg, pol = R.SolverConfig(mode="yx", nonmonotone=False), R.FixedRestart(50)
    fused = R.run_restarted(inst, cfg, pol, budget=150, criteria=crit(1e-9))
    emu = EmulatedCluster(world).run(
        inst, lambda sh: R.run_restarted(inst, cfg, pol, budget=150, criteria=crit(1e-9), shard=sh))
    for r in range(world):
        tr = np.load(tmp_path / f"{kind}{r}_trace.npy")
        x = np.load(tmp_path / f"{kind}{r}_x.npy")
        lam = np.load(tmp_path / f"{kind}{r}_lam.npy")
        np.testing.assert_array_equal(tr[:, TAU], trace_arr(fused.trace)[:, TAU])
        np.testing.assert_array_equal(tr, trace_arr(emu[r].trace)[:, :7])
        np.testing.assert_array_equal(x, emu[r].solution.x)
        np.testing.assert_array_equal(lam, emu[r].solution.lam)
        assert rel(x, fused.solution.x) <= 1e-12
