#!/bin/bash
# HYBRID at GPT-30B width: copy-engine vs SM-pull reduce-scatter + SM all-reduce (no staging round trip)
O=gpurun_out/${OUT:-r2hybsm}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in a b; do
  timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 > $O/hyb30_ce_$rep.json 2>/dev/null
  timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --rs-engine sm --rs-ctas 64 > $O/hyb30_sm_$rep.json 2>/dev/null
done
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --exposed > $O/t5_n4_auto.json 2>/dev/null
echo done
