#!/bin/bash
# Round 2: shared-GPU multi-rank parity (W ranks time-sharing cuda:0) + GPU suite + short bench.
set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.log 2>&1
for W in 2 4 8; do
  T0=$(date +%s)
  timeout 1200 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "parity and $W" > gpurun_out/r2a/mp_w$W.log 2>&1
  echo "W=$W rc=$? secs=$(( $(date +%s) - T0 ))" >> gpurun_out/r2a/mp_times.txt
done
timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu -k verify > gpurun_out/r2a/mp_verify.log 2>&1
echo "verify rc=$?" >> gpurun_out/r2a/mp_times.txt
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_multigpu.py > gpurun_out/r2a/pytest_gpu.log 2>&1
echo "suite rc=$?" >> gpurun_out/r2a/mp_times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a/bench_n1.json 2> gpurun_out/r2a/bench_n1.err
echo done
