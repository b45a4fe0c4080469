#!/bin/bash
# the whole GPU suite + smoke on a 2-GPU box (ranks W = 4 / 8 share the two GPUs)
O=gpurun_out/${OUT:-r2g2suite}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/times.txt
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_n2.json 2> $O/bench_n2.err
echo "bench n2 rc=$?" >> $O/times.txt
