#!/bin/bash
# Final round-2 evidence on a 4-GPU box: real-mode multi-GPU parity, the
# scaling points N=1/2/4 (self-launched), the reference arm at N=1/4, T5-11B,
# GPT-30B-width HYBRID, the AG/RS sweep, and the DMA DRAM-bytes range probe.
O=gpurun_out/${OUT:-r2final_n4}; mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpus.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1800 python -m pytest tests/test_multigpu.py -q -m gpu > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
for N in 1 2 4; do
  timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 --exposed > $O/bench_n$N.json 2> $O/bench_n$N.err
  echo "bench n=$N rc=$?" >> $O/times.txt
done
timeout 900 python bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err
echo "ref n4 rc=$?" >> $O/times.txt
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --exposed > $O/bench_t5_11b_n4.json 2> $O/bench_t5_11b_n4.err
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --exposed > $O/bench_gpt30b_l12_hybrid2x2_n4.json 2> $O/bench_gpt30b_l12_hybrid2x2_n4.err
timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 10 --warmup 3 --exposed > $O/bench_gpt1.3b_hybrid2x2_n4.json 2> $O/bench_gpt1.3b_hybrid2x2_n4.err
FSDP_SWEEP_SIZES=1,16,64,128,256,1024,2048 timeout 1500 python bench.py --gpus 4 --mode sweep > $O/sweep_n4.json 2> $O/sweep_n4.err
echo "sweep rc=$?" >> $O/times.txt
for MB in 12.6 134; do
  timeout 600 ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --csv \
    python tools/ncu_dma_range.py $MB > $O/ncu_dma_range_${MB}mb.csv 2> $O/ncu_dma_range_${MB}mb.err
done
echo done
