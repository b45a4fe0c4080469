#!/bin/bash
# last 1-GPU confirmation of the final code: the driver's GPU suite, smoke, bench (with cpu_baseline), reference arm
O=gpurun_out/${OUT:-r2final3_g1}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "build rc=$?" >> $O/times.txt
T0=$(date +%s)
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/times.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err
echo "bench rc=$?" >> $O/times.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err
echo "ref rc=$?" >> $O/times.txt
