O=gpurun_out/hyb; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --exposed --no-cpu-baseline > $O/bench_hybrid2x2_n4.json 2> $O/h.err; echo "rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --strategy SHARD_GRAD_OP --exposed --no-cpu-baseline > $O/bench_sgo_n4.json 2> $O/s.err; echo "rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --strategy NO_SHARD --no-cpu-baseline > $O/bench_noshard_n4.json 2> $O/n.err; echo "rc=$?"
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), (d.get('exposed_comm') or {}).get('frac_of_step'), json.dumps(d.get('comm_stalls')), {k:(round(v['mean_ms'],3), v['count']) for k,v in d['kernels'].items()})"; done
tail -3 $O/*.err
