#!/bin/bash
# piece-major all-gather DMA A/B on the large-shard configs + its parity schedule
O=gpurun_out/${OUT:-r2agp}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
MP_SCENARIOS=ce_schedules timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29561 tests/mp_worker.py > $O/ce_schedules.log 2>&1
echo "ce_schedules rc=$?" >> $O/times.txt
for rep in a b; do
  timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 > $O/t5_default_$rep.json 2>/dev/null
  FSDP_CE_AG_PIECE=$((32<<20)) timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 > $O/t5_piece32_$rep.json 2>/dev/null
done
timeout 2400 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 2 > $O/g30_default.json 2>/dev/null
FSDP_CE_AG_PIECE=$((32<<20)) timeout 2400 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 2 > $O/g30_piece32.json 2>/dev/null
FSDP_CE_AG_PIECE=$((64<<20)) timeout 2400 python bench.py --gpus 4 --config gpt30b --micro 1 --steps 3 --warmup 2 > $O/g30_piece64.json 2>/dev/null
echo done
