#!/bin/bash
# Round 2: shared-GPU multi-rank parity (W ranks time-sharing cuda:0) + GPU suite + short bench.
O=gpurun_out/${OUT:-r2c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for W in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr 127.0.0.1 --master-port 2952$W tools/shared_probe.py > $O/probe_w$W.log 2>&1
done
for W in 2 4 8; do
  T0=$(date +%s)
  timeout 1500 python -m pytest tests/test_multigpu.py -x -q -m gpu -k "parity and $W" > $O/mp_w$W.log 2>&1
  echo "W=$W rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/mp_times.txt
done
T0=$(date +%s)
timeout 1500 python -m pytest tests/test_multigpu.py -q -m gpu -k "not parity" > $O/mp_cli.log 2>&1
echo "cli rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/mp_times.txt
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_multigpu.py > $O/pytest_gpu.log 2>&1
echo "suite rc=$?" >> $O/mp_times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo done
