"""Copy-engine reduce-scatter schedule sweep (torchrun, one process per GPU).

Each variant sets the FSDP_CE_* schedule knobs (read when a communicator
first uses the copy engines), creates its own communicator and times
`reduce_scatter_ce` at several sizes with CUDA events (20 iterations after 5
warm-up, max over ranks).  busbw = S (W-1)/W / t, S = unsharded bf16 bytes.

    torchrun --nproc-per-node 4 tools/rs_ce_sweep.py > rs_ce.json
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

VARIANTS = {
    "pull_p1": {"FSDP_CE_RS_PUSH": "0", "FSDP_CE_RS_PIPE_MIN": str(1 << 40)},
    "push_p1": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIPE_MIN": str(1 << 40)},
    "pull_uni4": {"FSDP_CE_RS_PUSH": "0", "FSDP_CE_RS_GEOM": "0", "FSDP_CE_RS_PIECES": "4"},
    "push_uni4": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_GEOM": "0", "FSDP_CE_RS_PIECES": "4"},
    "push_geo_4M": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_MIN_PIECE": str(4 << 20)},
    "push_geo_8M": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_MIN_PIECE": str(8 << 20)},
    "push_geo_2M": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_MIN_PIECE": str(2 << 20)},
    "pull_geo_4M": {"FSDP_CE_RS_PUSH": "0", "FSDP_CE_RS_MIN_PIECE": str(4 << 20)},
    # diagnostics: transfers only (results wrong), and the all-gather's DMA at the same size
    "push_p1_noreduce": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIPE_MIN": str(1 << 40), "FSDP_CE_RS_NOREDUCE": "1"},
    "pull_p1_noreduce": {"FSDP_CE_RS_PUSH": "0", "FSDP_CE_RS_PIPE_MIN": str(1 << 40), "FSDP_CE_RS_NOREDUCE": "1"},
    "push_geo_noreduce": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_NOREDUCE": "1"},
    "ag_ce": {"_AG": "1"},
    # SM TMA-pull reduce-scatter ring geometries (FSDP_RS_TMA_RING) x grid
    **{f"tma_r{r}_c{c}": {"_TMA": "1", "FSDP_RS_TMA_RING": str(r), "_CTAS": str(c)}
       for r in range(4) for c in (64, 128)},
    **{f"hyb_f{int(f * 100)}": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_SM_FRAC": str(f)}
       for f in (0.1, 0.2, 0.3, 0.4)},
    "push_geo_p3": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIECES": "3", "FSDP_CE_RS_MIN_PIECE": str(1 << 20)},
    "push_geo_p4": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIECES": "4", "FSDP_CE_RS_MIN_PIECE": str(1 << 20)},
    "push_geo_p5": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIECES": "5", "FSDP_CE_RS_MIN_PIECE": str(1 << 20)},
    # pipelining at unit sizes (GPT-1.3B block at W=4: 12.6 M-element chunks):
    # geometric pieces down to 8 / 4 M elements (16 / 8 MB per member piece)
    "push_geo_u8M": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIPE_MIN": str(8 << 20),
                     "FSDP_CE_RS_MIN_PIECE": str(4 << 20)},
    "push_geo_u4M": {"FSDP_CE_RS_PUSH": "1", "FSDP_CE_RS_PIPE_MIN": str(4 << 20),
                     "FSDP_CE_RS_MIN_PIECE": str(2 << 20)},
    "pull_uni_u8M": {"FSDP_CE_RS_PUSH": "0", "FSDP_CE_RS_GEOM": "0", "FSDP_CE_RS_PIECES": "4",
                     "FSDP_CE_RS_PIPE_MIN": str(8 << 20)},
}


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2304_11277_b200.comm import DeviceComm
    sizes = [int(x) for x in os.environ.get("RS_SIZES_MB", "64,256,1024,2048").split(",")]
    only = os.environ.get("RS_VARIANTS")
    names = only.split(",") if only else list(VARIANTS)
    dev = torch.device("cuda", local)
    out = {"world": world, "sizes_mb": sizes, "variants": {}}
    for name in names:
        saved = {k: os.environ.get(k) for k in VARIANTS[name]}
        os.environ.update(VARIANTS[name])
        maxb = max(sizes) << 20
        cm = DeviceComm.create(2 * maxb + (64 << 20), max_ctas=int(os.environ.get("_CTAS", "64")))
        src, stage = cm.alloc(maxb), cm.alloc(maxb)
        row = {}
        for mb in sizes:
            S = mb << 20
            n = S // 2 // world
            cm.view(src, n * world, torch.bfloat16).copy_(torch.randn(n * world, device=dev).to(torch.bfloat16))
            o = torch.empty(n, device=dev)

            sh = torch.randn(n, device=dev).to(torch.bfloat16)

            def fn():
                if os.environ.get("_AG"):
                    cm.all_gather_ce((world, 1), sh, stage)
                elif os.environ.get("_TMA"):
                    cm.reduce_scatter_pull((world, 1), src, torch.bfloat16, [o], postdiv=float(world), tma=True)
                else:
                    cm.reduce_scatter_ce((world, 1), src, torch.bfloat16, stage, o, postdiv=float(world))
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 20], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            row[mb] = round(S * (world - 1) / world / (t.item() * 1e-3) / 1e9, 1)
        torch.cuda.synchronize()
        assert cm.device_error() == 0
        cm.close()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        out["variants"][name] = row
        if rank == 0:
            print(name, row, file=sys.stderr, flush=True)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
