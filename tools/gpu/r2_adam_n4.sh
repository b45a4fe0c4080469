#!/bin/bash
# in-step Adam ring variants at N=4 (fp32 gradients, 329 M-element arena per rank)
O=gpurun_out/${OUT:-r2adam4}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for V in 0 1 4 5 0 1; do
  FSDP_ADAM_VARIANT=$V timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-exposed > $O/n4_v${V}_$(date +%s).json 2>/dev/null
done
