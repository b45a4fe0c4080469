# Closing validation of the round on one 4-GPU box: gpurun_out/final4/
O=gpurun_out/final4; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "n1 rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo "ref1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --exposed > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --impl reference > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err; echo "ref4 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --mode sweep > $O/sweep_n4.json 2> $O/sweep_n4.err; echo "sweep4 rc=$?"
for f in $O/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('n_gpus'), (d.get('roofline') or {}).get('frac'), (d.get('exposed_comm') or {}).get('frac_of_step'), (d.get('clocks') or {}).get('sm_mhz'))"; done
