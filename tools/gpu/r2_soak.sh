#!/bin/bash
# flakiness soak: the multi-rank and bench-replica tests three times on a 1-GPU box (shared mode)
O=gpurun_out/${OUT:-r2soak}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2 3; do
  T0=$(date +%s)
  timeout 1500 python -m pytest tests/test_multigpu.py tests/test_bench_gpu.py -q -m gpu > $O/mp_$i.log 2>&1
  echo "run $i rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
done
