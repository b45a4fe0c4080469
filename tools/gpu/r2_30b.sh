#!/bin/bash
# GPT-30B at full depth on 4 GPUs (FULL_SHARD F=4: the per-rank memory of HYBRID 4x2 on 8 GPUs)
O=gpurun_out/${OUT:-r2_30b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 2 --exposed > $O/bench_gpt30b_n4.json 2> $O/bench_gpt30b_n4.err
timeout 2400 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 2 --opt-split-geom off > $O/bench_gpt30b_n4_nogeom.json 2> $O/bench_gpt30b_n4_nogeom.err
echo done
