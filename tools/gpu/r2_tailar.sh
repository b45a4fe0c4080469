#!/bin/bash
# last unit's replica all-reduce as an SM tail kernel (tail_ar) A/B on 4 GPUs + multi-GPU parity
O=gpurun_out/${OUT:-r2tailar}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
for rep in 1 2; do
  for v in on off; do
    F=""; [ $v = off ] && F="--no-tail-ar"
    timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 \
      --steps 10 --warmup 3 --no-cpu-baseline --check-replicas $F > $O/bench_hyb30b_${v}_$rep.json 2> $O/bench_hyb30b_${v}_$rep.err
    echo "hyb30b $v $rep rc=$?" >> $O/times.txt
  done
done
for v in on off; do
  F=""; [ $v = off ] && F="--no-tail-ar"
  timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 20 --warmup 5 \
    --no-cpu-baseline $F > $O/bench_hyb13b_$v.json 2> $O/bench_hyb13b_$v.err
  echo "hyb13b $v rc=$?" >> $O/times.txt
  timeout 900 python bench.py --gpus 4 --strategy NO_SHARD --steps 20 --warmup 5 \
    --no-cpu-baseline $F > $O/bench_noshard_$v.json 2> $O/bench_noshard_$v.err
  echo "noshard $v rc=$?" >> $O/times.txt
done
