"""Host-side checks of the in-kernel NVLink exchange (solver_ops.cuh:
peer_exchange, sharding.Shard.attach_peer_exchange) on the CPU:

* the protocol itself, modelled with R processes over shared memory: each
  "rank" pushes its partial into slot `rank` of set (gen & 1) of every peer's
  region, publishes generation `gen` in flag `rank` of every peer, waits for
  all R flags of its own region to reach `gen`, and sums its slots in rank
  order.  With random skews between ranks every rank must obtain the exact
  rank-ordered sum at every generation -- i.e. double buffering by generation
  parity is enough (a rank can be at most one exchange ahead);
* the IPC handshake over torch.distributed (gloo, world size 2) with the CUDA
  IPC calls mocked: the pointer table each rank registers has its own region
  at index rank and the opened peer regions elsewhere, in rank order."""

import multiprocessing as mpc
import os
import random
import socket
import time

import numpy as np
import pytest


def _rank_proc(rank, R, S, G, slots, flags, out):
    rng = random.Random(rank * 7919)
    slot = np.frombuffer(slots, dtype=np.float64).reshape(R, 2, R, S)     # [owner][set][writer][S]
    flag = np.frombuffer(flags, dtype=np.int64).reshape(R, R)             # [owner][writer]
    bad = 0
    for gen in range(1, G + 1):
        part = np.array([gen * 1000.0 + rank * 10.0 + k for k in range(S)])
        if rng.random() < 0.3:
            time.sleep(rng.random() * 0.002)              # skew
        st = gen & 1
        for peer in range(R):
            slot[peer, st, rank, :] = part
        for peer in range(R):
            flag[peer, rank] = gen                         # release (after the stores)
        for w in range(R):
            while flag[rank, w] < gen:                     # acquire
                time.sleep(0.0)
        total = slot[rank, st, 0, :].copy()
        for w in range(1, R):
            total = total + slot[rank, st, w, :]
        expect = sum(np.array([gen * 1000.0 + w * 10.0 + k for k in range(S)]) for w in range(R))
        bad += int(not np.array_equal(total, expect))
    out[rank] = bad


@pytest.mark.parametrize("R", [2, 3])
def test_peer_protocol_double_buffering(R):
    S, G = 4, 300
    ctx = mpc.get_context("fork")
    slots = ctx.RawArray("d", R * 2 * R * S)
    flags = ctx.RawArray("q", R * R)
    out = ctx.Array("i", R)
    procs = [ctx.Process(target=_rank_proc, args=(r, R, S, G, slots, flags, out)) for r in range(R)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert list(out) == [0] * R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _handshake_worker(rank, world, port, res):
    import torch.distributed as dist
    from paper_2605_29291_b200 import _capi
    from paper_2605_29291_b200.sharding import Shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeRegion:
        def __init__(self, nbytes):
            self.ptr = 1_000_000 * (rank + 1)

    _capi.PeerRegion = FakeRegion
    _capi.ipc_handle = lambda p: b"h" + str(p).encode()
    _capi.ipc_open = lambda h: int(h[1:].decode()) + 7      # "mapped" address of the peer region

    class Ctx:
        def peer_region_bytes(self):
            return 4096

        def set_peer_exchange(self, ptrs):
            self.ptrs = list(ptrs)

    try:
        shard = Shard(rank=rank, nranks=world, k0=0, k1=1, p2p=True)
        c = Ctx()
        shard.attach_peer_exchange(c)
        res[rank] = c.ptrs
    finally:
        dist.destroy_process_group()


def test_attach_peer_exchange_handshake_gloo():
    import torch.multiprocessing as tmp
    world = 2
    with tmp.Manager() as mgr:
        res = mgr.dict()
        tmp.spawn(_handshake_worker, args=(world, _free_port(), res), nprocs=world, join=True)
        got = dict(res)
    assert got[0] == [1_000_000, 2_000_007]
    assert got[1] == [1_000_007, 2_000_000]
