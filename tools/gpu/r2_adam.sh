#!/bin/bash
# in-step Adam ring geometry A/B at N=1 (bf16 and fp32 gradient arenas)
O=gpurun_out/${OUT:-r2adam}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for V in 0 5 6 7 8 5 6; do
  FSDP_ADAM_VARIANT=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bf16g_v${V}_$(date +%s).json 2>/dev/null
done
for V in 0 6 7; do
  FSDP_ADAM_VARIANT=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-w1-bf16-grad > $O/fp32g_v${V}_$(date +%s).json 2>/dev/null
done
echo done
