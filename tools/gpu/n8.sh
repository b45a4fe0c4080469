#!/bin/bash
# The N = 8 measurements of BASELINE.json's configs on one 8 x B200 node
# (gpurun offers at most 4 GPUs per call; this is what an 8-GPU box runs).
# Every command prints one JSON line; outputs land in gpurun_out/n8/.
set -x
O=gpurun_out/n8; mkdir -p $O
# 1. multi-rank parity on 8 real GPUs (IPC, copy engines, NVLS, every strategy incl. HYBRID 4x2 / 2x4)
timeout 2400 python -m pytest tests/test_multigpu.py -x -q -m gpu > $O/pytest_multigpu.log 2>&1
# 2. GPT-1.3B FULL_SHARD, the scaling points 1/2/4/8 (configs[1])
for N in 1 2 4 8; do
  timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --exposed > $O/bench_gpt1.3b_n$N.json 2> $O/bench_gpt1.3b_n$N.err
done
# 3. T5-11B FULL_SHARD, BACKWARD_PRE + limiter (configs[2])
timeout 1500 python bench.py --gpus 8 --config t5-11b --steps 6 --warmup 3 --exposed > $O/bench_t5_11b_n8.json 2> $O/bench_t5_11b_n8.err
# 4. GPT-30B HYBRID_SHARD 4 x 2 with sharded Adam (configs[3]); and 2 x 4
timeout 2400 python bench.py --gpus 8 --config gpt30b --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 4 --steps 4 --warmup 3 --exposed > $O/bench_gpt30b_hybrid4x2_n8.json 2> $O/bench_gpt30b_hybrid4x2_n8.err
timeout 2400 python bench.py --gpus 8 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 > $O/bench_gpt30b_l12_hybrid2x4_n8.json 2> $O/bench_gpt30b_l12_hybrid2x4_n8.err
# 5. AG/RS sweep 1 MB - 2 GB vs NCCL (configs[4])
timeout 1800 python bench.py --gpus 8 --mode sweep > $O/sweep_n8.json 2> $O/sweep_n8.err
# 6. the reference arm at N = 8 (CPU, shardsim algorithm)
timeout 1200 python bench.py --impl reference --gpus 8 --steps 1 --warmup 1 > $O/bench_ref_n8.json 2> $O/bench_ref_n8.err
