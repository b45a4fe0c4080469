#!/bin/bash
# GPT-30B width HYBRID 4 x 2 (the configs[3] communication pattern at full unit size: reduce-scatter
# over 4, replica all-reduce over pairs {r, r+4} of 154 M-element fp32 shards) with 8 ranks on a
# 4-GPU box (two ranks time-sharing each GPU: a correctness-at-size run, not a speed number)
O=gpurun_out/${OUT:-r2hyb42}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29571 \
  bench.py --gpus 8 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 4 --steps 2 --warmup 1 \
  --no-exposed --no-cpu-baseline > $O/bench_hybrid4x2_8ranks.json 2> $O/bench_hybrid4x2_8ranks.err
echo "rc=$?" > $O/rc.txt
nvidia-smi --query-gpu=index,memory.used --format=csv >> $O/rc.txt 2>&1
