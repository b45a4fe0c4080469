#!/bin/bash
# end-of-round confirmation on 4 GPUs, final code: real-mode parity, GPT-1.3B N = 1 / 2 / 4,
# T5-11B, GPT-30B width HYBRID 2 x 2 (default bf16 stage 2) vs the NCCL backend
O=gpurun_out/${OUT:-r2final3_n4}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 1800 python -m pytest tests/test_multigpu.py tests/test_bench_gpu.py -q -m gpu > $O/pytest_multigpu.log 2>&1
echo "multigpu rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
echo "n1 rc=$?" >> $O/times.txt
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.json 2> $O/bench_n2.err
echo "n2 rc=$?" >> $O/times.txt
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --exposed > $O/bench_n4.json 2> $O/bench_n4.err
echo "n4 rc=$?" >> $O/times.txt
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --exposed > $O/bench_t5_11b_n4.json 2> $O/bench_t5_11b_n4.err
echo "t5 rc=$?" >> $O/times.txt
timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --strategy HYBRID_SHARD --hybrid-shard-size 2 \
  --steps 10 --warmup 3 --no-cpu-baseline --check-replicas > $O/bench_gpt30b_l12_hyb2x2.json 2> $O/bench_gpt30b_l12_hyb2x2.err
echo "30b hyb rc=$?" >> $O/times.txt
timeout 900 python bench.py --gpus 4 --config gpt30b-l12 --micro 1 --backend nccl --strategy HYBRID_SHARD \
  --hybrid-shard-size 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gpt30b_l12_hyb2x2_nccl.json 2> $O/bench_gpt30b_l12_hyb2x2_nccl.err
echo "30b nccl rc=$?" >> $O/times.txt
