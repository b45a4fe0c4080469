#!/bin/bash
# Final round-2 evidence on a 1-GPU box: the driver's GPU suite + smoke, the
# default bench line, its ncu launch list, and one ncu --set full of the dominant kernel.
O=gpurun_out/${OUT:-r2final_g1}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T0=$(date +%s)
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/times.txt
T0=$(date +%s)
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err
echo "bench rc=$? secs=$(( $(date +%s) - T0 ))" >> $O/times.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err
echo "ref rc=$?" >> $O/times.txt
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_n1.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $O/times.txt
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:adam_tma --launch-count 1 \
  -o $O/ncu_adam_n1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_adam.log 2>&1
echo "ncu adam rc=$?" >> $O/times.txt
echo done
