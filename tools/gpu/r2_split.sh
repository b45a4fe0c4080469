#!/bin/bash
# A/B: optimizer launches at doubling unit counts (opt_split_geom) vs the 2-launch split
O=gpurun_out/${OUT:-r2split}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in a b; do
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > $O/gpt_n4_default_$rep.json 2>/dev/null
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --opt-split-geom --opt-split-first 1 > $O/gpt_n4_geom_$rep.json 2>/dev/null
done
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 > $O/t5_n4_default.json 2>/dev/null
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --opt-split-geom --opt-split-first 1 > $O/t5_n4_geom.json 2>/dev/null
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 > $O/t5_n4_default_b.json 2>/dev/null
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --opt-split-geom --opt-split-first 1 > $O/t5_n4_geom_b.json 2>/dev/null
echo done
