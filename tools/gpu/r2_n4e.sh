#!/bin/bash
# same-box A/B: in-place replica all-reduce (pool arena) and the W=1 bf16 gradient arena;
# GPU tests of the new kernels; DMA DRAM bytes by ncu range replay; ncu capture of the bf16-grad Adam.
O=gpurun_out/${OUT:-r2n4e}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py tests/test_session.py -q -m gpu > $O/pytest_kernels_runtime.log 2>&1
echo "pytest rc=$?" >> $O/times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/times.txt
for rep in a b; do
  timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 10 --warmup 3 --exposed > $O/hyb13_pool_$rep.json 2> /dev/null
  timeout 900 python bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 10 --warmup 3 --exposed --no-ar-pool > $O/hyb13_nopool_$rep.json 2> /dev/null
done
timeout 900 python bench.py --gpus 4 --strategy NO_SHARD --steps 10 --warmup 3 > $O/noshard_pool.json 2> /dev/null
timeout 900 python bench.py --gpus 4 --strategy NO_SHARD --steps 10 --warmup 3 --no-ar-pool > $O/noshard_nopool.json 2> /dev/null
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 > $O/hyb30_pool.json 2> /dev/null
timeout 1500 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 --steps 4 --warmup 3 --no-ar-pool > $O/hyb30_nopool.json 2> /dev/null
for MB in 12.6 25 134; do
  timeout 600 ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --csv \
    python tools/ncu_dma_range.py $MB > $O/ncu_dma_range_${MB}mb.csv 2> $O/ncu_dma_range_${MB}mb.err
done
export CUDA_VISIBLE_DEVICES=0
for rep in a b; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/n1_bf16g_$rep.json 2> /dev/null
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-w1-bf16-grad > $O/n1_fp32g_$rep.json 2> /dev/null
done
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:adam_tma --launch-count 1 \
  -o $O/ncu_adam_bf16g_n1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_adam.log 2>&1
echo done
