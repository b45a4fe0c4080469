# Round-end validation on one 4-GPU box: every result lands in gpurun_out/final2/
O=gpurun_out/final2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpus.csv
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "n1 rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo "ref1 rc=$?"
timeout 900 python bench.py --impl torch-unsharded > $O/bench_torch_unsharded_n1.json 2> $O/bench_tu.err; echo "tu rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --exposed > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --impl reference > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err; echo "ref4 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --config t5-11b --steps 6 --exposed --no-cpu-baseline > $O/bench_t5_11b_n4.json 2> $O/bench_t5.err; echo "t5 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --config gpt30b --micro 1 --steps 4 --no-cpu-baseline > $O/bench_gpt30b_n4.json 2> $O/bench_gpt30b.err; echo "30b rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29606 bench.py --gpus 4 --mode sweep > $O/sweep_n4.json 2> $O/sweep_n4.err; echo "sweep4 rc=$?"
timeout 1200 $TR --nproc-per-node 2 --master-port 29607 bench.py --gpus 2 --mode sweep > $O/sweep_n2.json 2> $O/sweep_n2.err; echo "sweep2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adam_tma --launch-skip 2 --launch-count 1 -f -o $O/ncu_adam_default python tools/adam_bench.py --one 1315819520 > $O/ncu_adam.log 2>&1; echo "ncu rc=$?"
for f in $O/bench_*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('n_gpus'), (d.get('roofline') or {}).get('frac'), (d.get('exposed_comm') or {}).get('frac_of_step'))
except Exception as e: print('$f', 'ERR', e)"; done
