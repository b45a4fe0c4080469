#!/bin/bash
# Debug shared-GPU timeouts: session parity at W=2, verify at W=2, plus a barrier-latency probe.
mkdir -p gpurun_out/r2b
cat > /tmp/probe.py <<'PY'
import os, time, torch, torch.distributed as dist
from paper_2304_11277_b200.dist_util import init_from_env
from paper_2304_11277_b200.comm import DeviceComm
rank, world, dev = init_from_env()
c = DeviceComm.create(64 << 20)
a, b = c.alloc(8 << 20), c.alloc(8 << 20)
x = torch.ones(1024, device="cuda", dtype=torch.bfloat16)
out = torch.empty(2048, device="cuda")
for name, fn in (("ag_ce", lambda: c.all_gather_ce((world, 1), x, a)),
                 ("ar_ce", lambda: c.all_reduce_ce((world, 1), x, a, b, out)),
                 ("ag_sm", lambda: c.all_gather((world, 1), [x], a, torch.bfloat16))):
    torch.cuda.synchronize(); dist.barrier()
    t = time.time()
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    dt = (time.time() - t) / 50
    if rank == 0:
        print(f"{name}: {dt*1e3:.3f} ms/call err={c.device_error()}", flush=True)
c.close()
PY
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 /tmp/probe.py > gpurun_out/r2b/probe_w2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 /tmp/probe.py > gpurun_out/r2b/probe_w4.log 2>&1
MP_SCENARIOS=session_parity timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29513 tests/mp_worker.py > gpurun_out/r2b/session_w2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29514 -m paper_2304_11277_b200 verify --steps 3 > gpurun_out/r2b/verify_w2.log 2>&1
MP_SCENARIOS=fsdp_step timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29515 tests/mp_worker.py > gpurun_out/r2b/steps_w2.log 2>&1
echo done
