"""Per-call latency of the IPC collectives when W ranks share one GPU
(time-sliced contexts) or own one GPU each: torchrun --nproc-per-node W tools/shared_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2304_11277_b200.comm import DeviceComm  # noqa: E402
from paper_2304_11277_b200.dist_util import init_from_env, shared_gpu  # noqa: E402

rank, world, dev = init_from_env()
c = DeviceComm.create(64 << 20)
a, b = c.alloc(8 << 20), c.alloc(8 << 20)
ll = c.alloc(c.ll_bytes(world, 1024, torch.bfloat16), 16)
x = torch.ones(1024, device="cuda", dtype=torch.bfloat16)
out = torch.empty(1024 * world, device="cuda")
for name, fn in (("ag_ce", lambda: c.all_gather_ce((world, 1), x, a)),
                 ("ar_ce", lambda: c.all_reduce_ce((world, 1), x, a, b, out)),
                 ("ag_sm", lambda: c.all_gather((world, 1), [x], a, torch.bfloat16)),
                 ("ag_ll", lambda: c.all_gather_ll((world, 1), [x], a, torch.bfloat16, ll))):
    torch.cuda.synchronize()
    dist.barrier()
    t = time.time()
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    dt = (time.time() - t) / 50
    if rank == 0:
        print(f"W={world} shared={shared_gpu(world)} {name}: {dt * 1e3:.3f} ms/call err={c.device_error()}",
              flush=True)
c.close()
