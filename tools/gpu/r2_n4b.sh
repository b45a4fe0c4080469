#!/bin/bash
# HYBRID stage 2 on its own stream (A/B vs profiles/r2/n4_a), DMA per-copy cost,
# CE reduce-scatter piece schedules at unit sizes, ncu DRAM bytes of ce_reduce.
O=gpurun_out/${OUT:-r2n4b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/dma_probe.py > $O/dma_probe.json 2> $O/dma_probe.err
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --exposed > $O/bench_gpt30b_l12_hybrid2x2_n4.json 2> $O/bench_gpt30b_l12_hybrid2x2_n4.err
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 2 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --exposed > $O/bench_gpt30b_l12_hybrid2x2_n4_micro2.json 2> $O/bench_gpt30b_l12_hybrid2x2_n4_micro2.err
timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 10 --warmup 3 --exposed > $O/bench_gpt1.3b_hybrid2x2_n4.json 2> $O/bench_gpt1.3b_hybrid2x2_n4.err
# CE reduce-scatter schedules at the in-step unit sizes (GPT-1.3B block 100 MB, T5 decoder 537 MB) and 2 GiB
RS_SIZES_MB=100,256,537,2048 RS_VARIANTS=pull_p1,push_p1,pull_uni4,push_uni4,push_geo_2M,push_geo_p3,push_geo_p4,push_p1_noreduce,pull_p1_noreduce,ag_ce \
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29531 tools/rs_ce_sweep.py > $O/rs_ce_n4.json 2> $O/rs_ce_n4.err
# ncu: DRAM bytes of the copy-engine reduction kernel (local, never waits: safe to replay) at W=2, 100 MB
RS_SIZES_MB=100 RS_VARIANTS=pull_p1 timeout 900 ncu --target-processes all --kernel-name regex:ce_reduce --launch-count 2 \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29532 tools/rs_ce_sweep.py > $O/ncu_ce_reduce_w2.csv 2> $O/ncu_ce_reduce_w2.err
echo done
