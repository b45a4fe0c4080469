O=gpurun_out/t5rs; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "--rs-engine ce" "--rs-engine sm --rs-ctas 32" "--rs-engine sm --rs-ctas 64" "--rs-engine ce"; do
i=$((i+1))
timeout 1200 $TR --nproc-per-node 4 --master-port 2990$i bench.py --gpus 4 --config t5-11b --steps 6 --exposed --no-cpu-baseline $cfg > $O/t5_$i.json 2> $O/t5_$i.err
python -c "
import json
d=json.loads(open('$O/t5_$i.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']/d['n_gpus'],1), (d.get('exposed_comm') or {}).get('frac_of_step'), d['clocks']['sm_mhz'], (d.get('exposed_comm') or {}).get('rank_compute_spread',{}).get('spread_ms'))" || tail -3 $O/t5_$i.err
done
