#!/bin/bash
# pool-resident gradient arena for HYBRID/NO_SHARD (all-reduce lands in place),
# real-mode parity at W=2/4, HYBRID benches incl. the NCCL comparison, DMA DRAM bytes by ncu range replay.
O=gpurun_out/${OUT:-r2n4d}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1800 python -m pytest tests/test_multigpu.py -q -m gpu -x > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --exposed > $O/bench_gpt30b_l12_hybrid2x2_n4.json 2> $O/bench_gpt30b_l12_hybrid2x2_n4.err
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --backend nccl > $O/bench_gpt30b_l12_hybrid2x2_n4_nccl.json 2> $O/bench_gpt30b_l12_hybrid2x2_n4_nccl.err
timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 10 --warmup 3 --exposed > $O/bench_gpt1.3b_hybrid2x2_n4.json 2> $O/bench_gpt1.3b_hybrid2x2_n4.err
timeout 900 python bench.py --gpus 4 --strategy NO_SHARD --steps 10 --warmup 3 --exposed > $O/bench_gpt1.3b_noshard_n4.json 2> $O/bench_gpt1.3b_noshard_n4.err
for MB in 12.6 25 134; do
  timeout 600 ncu --replay-mode range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --csv \
    python tools/ncu_dma_range.py $MB > $O/ncu_dma_range_${MB}mb.csv 2> $O/ncu_dma_range_${MB}mb.err
done
echo done
