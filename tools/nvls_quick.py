"""Quick NVLS check under torchrun: tests/mp_worker.nvls_collectives plus a
bandwidth comparison of the multicast vs unicast all-gather at 256 MB."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    import mp_worker
    res = {}
    mp_worker.nvls_collectives(rank, world, res)
    from paper_2304_11277_b200.comm import DeviceComm
    for ctas in (8, 16, 32):
        cm = DeviceComm.create(1 << 30, max_ctas=ctas, nvls_group=world)
        off = cm.alloc(512 << 20)
        S = 256 << 20
        n = S // 2 // world
        x = torch.randn(n, device="cuda").to(torch.bfloat16)
        for name, fn in (("nvls", lambda: cm.all_gather_nvls((world, 1), x, off, torch.bfloat16)),
                         ("sm", lambda: cm.all_gather((world, 1), [x], off, torch.bfloat16))):
            for _ in range(5):
                fn()
            torch.cuda.synchronize(); dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record(); torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 20], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[f"{name}_c{ctas}_gbs"] = round(S * (world - 1) / world / (t.item() * 1e-3) / 1e9, 1)
        cm.close()
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
