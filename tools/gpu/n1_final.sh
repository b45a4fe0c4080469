set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adam_tma --launch-skip 2 --launch-count 1 -f -o gpurun_out/ncu_adam6144 python tools/adam_bench.py --one 1315819520 > gpurun_out/ncu_adam6144.log 2>&1; tail -3 gpurun_out/ncu_adam6144.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -3 gpurun_out/ncu_launch.log
