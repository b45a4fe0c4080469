#!/bin/bash
# 8 ranks on a 4-GPU box (two ranks time-sharing each GPU; correctness at size, not speed numbers):
#  - GPT-30B width HYBRID 4 x 2 (configs[3]'s pattern at full unit size: reduce-scatter over 4,
#    replica all-reduce over pairs {r, r+4} of 154 M-element fp32 shards), replica digests checked
#  - GPT-30B width HYBRID 2 x 4 (8 layers), replica digests checked
#  - GPT-1.3B FULL_SHARD F = 8
# then the self-launched 4-GPU bench (one rank per GPU)
O=gpurun_out/${OUT:-r2hyb42}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run8() {  # name, args...
  local n=$1; shift
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 \
    --master-port 29571 bench.py --gpus 8 "$@" > $O/$n.json 2> $O/$n.err
  echo "$n rc=$?" >> $O/rc.txt
}
run8 hybrid4x2_gpt30b_l12 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 4 \
  --steps 5 --warmup 3 --no-exposed --no-cpu-baseline --check-replicas
run8 hybrid2x4_gpt30b_l8 --config gpt30b-l8 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 \
  --steps 3 --warmup 3 --no-exposed --no-cpu-baseline --check-replicas
run8 full8_gpt13b --config gpt1.3b --micro 4 --steps 5 --warmup 3 --no-exposed --no-cpu-baseline
timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n4.json 2> $O/bench_n4.err
echo "bench_n4 rc=$?" >> $O/rc.txt
nvidia-smi --query-gpu=index,memory.used --format=csv >> $O/rc.txt 2>&1
