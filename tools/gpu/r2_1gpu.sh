#!/bin/bash
# 1-GPU box: the full GPU suite as the driver runs it (multi-rank tests in shared mode),
# smoke, and the in-step Adam ring variants with the bf16-gradient arena.
O=gpurun_out/${OUT:-r2g1}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/times.txt
for V in 0 3 4 5 0; do
  FSDP_ADAM_VARIANT=$V timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/n1_adam_v$V.json 2>/dev/null
  cp $O/n1_adam_v$V.json $O/n1_adam_v${V}_$(date +%s).json
done
echo done
