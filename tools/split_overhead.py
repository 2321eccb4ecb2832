"""Cost of one exchange round trip in split (sharded) mode on ONE GPU:
C1 solve fused vs forced-split with (a) a no-op exchange, (b) torch
all_reduce over NCCL (world size 1)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from paper_2605_29291_b200.sharding import Shard  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
arr = instances.config_instance(name)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
cfg = R.SolverConfig(mode="yx", nonmonotone=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
calls = [0]


def noop(views):
    calls[0] += 1


def nccl(views):
    calls[0] += 1
    for v in views:
        dist.all_reduce(v)


for label, shard in [("fused", None),
                     ("split-noop", Shard(0, 1, 0, arr.m + 1, exchange=noop, force_split=True)),
                     ("split-nccl", Shard(0, 1, 0, arr.m + 1, exchange=nccl, force_split=True)),
                     ("peer-p2p", Shard(0, 1, 0, arr.m + 1, exchange=nccl, force_split=True, p2p=True))]:
    for rep in range(2):
        calls[0] = 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = R.run_restarted(inst, cfg, R.FixedRestart(500), budget=50_000, criteria=crit, shard=shard)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{label:11s} {dt * 1e3:8.1f} ms  {res.iterations} it  {calls[0]} exchanges  "
          f"{res.device_stats['run_launches']} run calls")
dist.destroy_process_group()
