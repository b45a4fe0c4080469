#!/bin/bash
# final-code confirmation on 4 GPUs: real-mode parity, GPT-1.3B N=4, T5-11B with the auto piece-major gather
O=gpurun_out/${OUT:-r2final2_n4}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1800 python -m pytest tests/test_multigpu.py -q -m gpu > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --exposed > $O/bench_n4.json 2> $O/bench_n4.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --exposed > $O/bench_t5_11b_n4.json 2> $O/bench_t5_11b_n4.err
FSDP_CE_AG_PIECE=0 timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 > $O/bench_t5_11b_n4_nopiece.json 2> /dev/null
for MB in 134; do
  timeout 600 ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --csv \
    python tools/ncu_dma_range.py $MB 32 > $O/ncu_dma_range_${MB}mb_piece32.csv 2> /dev/null
done
echo done
