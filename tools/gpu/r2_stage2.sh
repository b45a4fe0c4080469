#!/bin/bash
# HYBRID stage-2 payload A/B (fp32 partials vs the reduce dtype) on 4 GPUs + the multi-GPU parity
O=gpurun_out/${OUT:-r2stage2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "build rc=$?" >> $O/times.txt
T0=$(date +%s)
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
for rep in 1 2; do
  for s2 in fp32 reduce; do
    timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 \
      --hybrid-stage2 $s2 --steps 10 --warmup 3 --no-cpu-baseline --check-replicas \
      > $O/bench_gpt30b_l12_hyb2x2_${s2}_$rep.json 2> $O/bench_gpt30b_l12_hyb2x2_${s2}_$rep.err
    echo "30b $s2 $rep rc=$?" >> $O/times.txt
  done
done
for s2 in fp32 reduce; do
  timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --hybrid-stage2 $s2 \
    --steps 10 --warmup 3 --no-cpu-baseline --check-replicas > $O/bench_gpt13b_hyb2x2_${s2}.json 2> $O/bench_gpt13b_hyb2x2_${s2}.err
  echo "1.3b $s2 rc=$?" >> $O/times.txt
done
timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --backend nccl --strategy HYBRID_SHARD \
  --hybrid-shard-size 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gpt30b_l12_hyb2x2_nccl.json 2> $O/bench_gpt30b_l12_hyb2x2_nccl.err
echo "30b nccl rc=$?" >> $O/times.txt
