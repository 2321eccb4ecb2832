"""Constraint sharding across GPUs.

Rank r holds matrices ``[k0, k1)`` of the m+1 quadratic forms (Q_0 counts as
rank 0's work); x, the multipliers and all vectors are replicated.  Every
backtracking trial exchanges (all-reduce, sum) one n-vector -- this rank's
share of ``sum_i w_i (u_i + q_i)`` -- and one (m+1)-vector of constraint values
(exact: disjoint supports); the accept/reject decision is then computed
identically on every rank, so the host control flow stays in lockstep without
further communication.  The smoothed gap adds one exchange of H (n x n) per
adaptive check.

* ``nccl_shard(inst)``: the production path -- one process per GPU; the
  library owns an NCCL communicator (``_capi.Comm``, bootstrapped once per
  process from a unique id that rank 0 broadcasts over ``torch.distributed``)
  and sums every exchange itself, rank-ordered (csrc/comm.cuh), without a
  host callback: NCCL moves the bytes over NVLink/NVSwitch, the sum order is
  fixed, so every rank and every algorithm NCCL picks give the
  same bits.
* ``group_shard(inst, group)``: the same rank-ordered exchange through a
  ``torch.distributed`` group at the host (any backend, e.g. gloo): used to
  run real multi-process shards where NCCL cannot (several ranks on one GPU:
  the kernels stop at every exchange point, so they never wait on each other).
* ``EmulatedCluster``: R shards of one instance on ONE GPU, driven by R host
  threads that meet at each exchange (the kernels never wait on each other:
  each launch ends at the exchange point).  Used by the tests.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class Shard:
    rank: int
    nranks: int
    k0: int
    k1: int
    exchange: Optional[Callable[[list], None]] = None   # all-reduce(sum) of a list of device tensors
    force_split: bool = False
    name: str = ""
    l0: Optional[int] = None      # factored instances: linear rows [l0, l1) of this rank
    l1: Optional[int] = None
    p2p: bool = False             # dense: exchange in-kernel over NVLink peer memory (opt-in)
    group: object = None          # torch.distributed group for the peer-region handshake
    comm: object = None           # _capi.Comm: native rank-ordered NCCL exchange (no host callback)
    _peer: object = None          # [(region, opened peer pointers)] kept alive by the shard

    def attach_peer_exchange(self, ctx):
        """Allocate this rank's zeroed exchange region, swap CUDA IPC handles
        with the other ranks (torch.distributed object all-gather) and hand the
        R pointers to the context (rapdb_set_peer_exchange)."""
        from . import _capi
        region = _capi.PeerRegion(ctx.peer_region_bytes())
        if self.nranks == 1:
            ptrs = [region.ptr]
            opened = []
        else:
            import torch.distributed as dist
            allh = [None] * self.nranks
            dist.all_gather_object(allh, _capi.ipc_handle(region.ptr), group=self.group)
            ptrs, opened = [], []
            for r, hr in enumerate(allh):
                if r == self.rank:
                    ptrs.append(region.ptr)
                else:
                    p = _capi.ipc_open(hr)
                    opened.append(p)
                    ptrs.append(p)
            dist.barrier(group=self.group)
        ctx.set_peer_exchange(ptrs)
        # every engine gets a fresh region (its flags restart at generation 0);
        # earlier regions stay mapped so engines created before remain valid
        if self._peer is None:
            self._peer = []
        self._peer.append((region, opened))

    @property
    def split(self) -> bool:
        return self.nranks > 1 or self.force_split


def plan(m: int, nranks: int, zero_flags: Optional[Sequence[bool]] = None) -> List[Tuple[int, int]]:
    """Contiguous ranges of the m+1 matrices, balanced by streamed (non-zero)
    matrices; every rank gets at least one matrix when m+1 >= nranks."""
    total = m + 1
    if nranks < 1 or nranks > total:
        raise ValueError(f"cannot shard {total} matrices over {nranks} ranks")
    cost = np.ones(total) if zero_flags is None else np.where(np.asarray(zero_flags, bool), 0.05, 1.0)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [0]
    for r in range(1, nranks):
        target = cum[-1] * r / nranks
        k = int(np.searchsorted(cum, target, side="left"))
        k = max(k, bounds[-1] + 1)
        k = min(k, total - (nranks - r))
        bounds.append(k)
    bounds.append(total)
    return [(bounds[r], bounds[r + 1]) for r in range(nranks)]


def shard_ranges(inst, nranks: int):
    """[(k0, k1, l0, l1)] per rank: matrix ranges balanced by streamed
    matrices (dense; l0 = l1 = None) or the factored instance's own plan."""
    if hasattr(inst, "shard_ranges"):
        return inst.shard_ranges(nranks)
    return [(k0, k1, None, None) for k0, k1 in plan(inst.m, nranks, inst.zero_flags().astype(bool))]


_COMMS = {}


def native_comm(group=None, device_index: Optional[int] = None):
    """The process's native NCCL communicator for a torch.distributed group
    (created once, collectively: rank 0 makes the unique id and broadcasts it
    over the group -- bootstrap only, no solver data goes through torch)."""
    import torch
    import torch.distributed as dist
    from . import _capi
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.cuda.current_device() if device_index is None else int(device_index)
    key = (id(group), world, rank, dev)
    if key not in _COMMS:
        box = [_capi.comm_unique_id() if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(box, src=src, group=group)
        _COMMS[key] = _capi.Comm(dev, box[0], rank, world)
    return _COMMS[key]


def nccl_shard(inst, group=None, device_index: Optional[int] = None) -> Shard:
    """This process's shard for the current torch.distributed group, with the
    library's own rank-ordered NCCL exchange."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    k0, k1, l0, l1 = shard_ranges(inst, world)[rank]
    return Shard(rank=rank, nranks=world, k0=k0, k1=k1, name="nccl", l0=l0, l1=l1, group=group,
                 comm=native_comm(group, device_index))


def ordered_allreduce_host(views, group=None):
    """Rank-ordered in-place sum of tensors across a torch.distributed group
    (any backend): all-gather the R contributions, then add them as
    ((p_0 + p_1) + p_2) + ... -- the association csrc/comm.cuh, the emulated
    cluster and the in-kernel peer exchange use.  CUDA tensors are staged
    through the host when the backend is gloo."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return
    host = dist.get_backend(group) == "gloo"
    for v in views:
        src = v.detach().to("cpu") if host and v.is_cuda else v.detach()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src.contiguous(), group=group)
        tot = parts[0].clone()
        for r in range(1, world):
            tot += parts[r]
        v.copy_(tot)
    if any(v.is_cuda for v in views):
        torch.cuda.synchronize()


def group_shard(inst, group=None) -> Shard:
    """This process's shard, exchanging through ``ordered_allreduce_host``
    over a torch.distributed group (multi-process runs on one GPU, gloo)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    k0, k1, l0, l1 = shard_ranges(inst, world)[rank]
    return Shard(rank=rank, nranks=world, k0=k0, k1=k1, name="group", l0=l0, l1=l1, group=group,
                 exchange=lambda views: ordered_allreduce_host(views, group), force_split=True)


class EmulatedCluster:
    """R shards on one GPU: one host thread per rank, a rank-ordered sum at each
    exchange (rank 0 adds the R buffers in rank order and writes the total back)."""

    def __init__(self, nranks: int):
        self.R = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots: List[Optional[list]] = [None] * nranks
        self.error: Optional[BaseException] = None

    def shards(self, inst) -> List[Shard]:
        out = []
        for r, (k0, k1, l0, l1) in enumerate(shard_ranges(inst, self.R)):
            out.append(Shard(rank=r, nranks=self.R, k0=k0, k1=k1, force_split=True, name="emulated",
                             exchange=(lambda views, rr=r: self._exchange(rr, views)), l0=l0, l1=l1))
        return out

    def _exchange(self, rank, views):
        import torch
        self.slots[rank] = views
        self.barrier.wait()
        if rank == 0:
            for i in range(len(views)):
                tot = self.slots[0][i].clone()
                for r in range(1, self.R):
                    tot += self.slots[r][i]
                for r in range(self.R):
                    self.slots[r][i].copy_(tot)
            torch.cuda.synchronize()
        self.barrier.wait()

    def run(self, inst, fn):
        """fn(shard) on every rank in parallel threads; returns the per-rank results."""
        shards = self.shards(inst)
        results: List = [None] * self.R
        errors: List = [None] * self.R

        def body(r):
            try:
                results[r] = fn(shards[r])
            except BaseException as exc:   # noqa: BLE001 -- re-raised below
                errors[r] = exc
                self.barrier.abort()

        threads = [threading.Thread(target=body, args=(r,)) for r in range(self.R)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errors:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in errors:
            if e is not None:
                raise e
        return results
