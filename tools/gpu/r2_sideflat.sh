#!/bin/bash
# gradient write-back on the reduce-scatter stream (side_flatten) A/B on 4 GPUs + multi-GPU parity
O=gpurun_out/${OUT:-r2sideflat}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
for v in on off; do
  F=""; [ $v = off ] && F="--no-side-flatten"
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline $F > $O/bench_n4_$v.json 2> $O/bench_n4_$v.err
  echo "n4 $v rc=$?" >> $O/times.txt
done
for v in on off; do
  F=""; [ $v = off ] && F="--no-side-flatten"
  timeout 1500 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 3 --no-cpu-baseline $F > $O/bench_gpt30b_$v.json 2> $O/bench_gpt30b_$v.err
  echo "30b $v rc=$?" >> $O/times.txt
  timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --no-cpu-baseline $F > $O/bench_t5_$v.json 2> $O/bench_t5_$v.err
  echo "t5 $v rc=$?" >> $O/times.txt
  timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 \
    --steps 10 --warmup 3 --no-cpu-baseline $F > $O/bench_hyb30b_$v.json 2> $O/bench_hyb30b_$v.err
  echo "hyb $v rc=$?" >> $O/times.txt
done
