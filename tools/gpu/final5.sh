O=gpurun_out/final5; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 $TR --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --config t5-11b --steps 6 --exposed --no-cpu-baseline > $O/bench_t5_11b_n4.json 2> $O/t5.err; echo "t5 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --config gpt30b --micro 1 --steps 4 --no-cpu-baseline > $O/bench_gpt30b_n4.json 2> $O/g30.err; echo "30b rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --exposed --no-cpu-baseline > $O/bench_hybrid2x2_n4.json 2> $O/h.err; echo "hyb rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --strategy NO_SHARD --exposed --no-cpu-baseline > $O/bench_noshard_n4.json 2> $O/n.err; echo "ns rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --strategy SHARD_GRAD_OP --exposed --no-cpu-baseline > $O/bench_sgo_n4.json 2> $O/s.err; echo "sgo rc=$?"
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), (d.get('exposed_comm') or {}).get('frac_of_step'), d['clocks']['sm_mhz'], d.get('peak_mem_gb'), d.get('num_alloc_retries'))"; done
