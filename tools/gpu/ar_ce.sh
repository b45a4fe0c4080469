O=gpurun_out/arce; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -3 $O/pytest_mgpu.log
timeout 900 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --strategy HYBRID_SHARD --hybrid-shard-size 2 --exposed --no-cpu-baseline > $O/bench_hybrid2x2_n4.json 2> $O/h.err; echo "rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --strategy NO_SHARD --exposed --no-cpu-baseline > $O/bench_noshard_n4.json 2> $O/n.err; echo "rc=$?"
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), (d.get('exposed_comm') or {}).get('frac_of_step'), json.dumps(d.get('comm_stalls')), {k:(round(v['mean_ms'],3), v['count']) for k,v in d['kernels'].items()})"; done
