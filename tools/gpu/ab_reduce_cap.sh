O=gpurun_out/cap; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cap in 0 148 48; do
i=$((i+1))
FSDP_CE_REDUCE_CAP=$cap timeout 1200 $TR --nproc-per-node 4 --master-port 2964$i bench.py --gpus 4 --config t5-11b --steps 6 --exposed --no-cpu-baseline > $O/t5_cap$cap.json 2>$O/t5_cap$cap.err
FSDP_CE_REDUCE_CAP=$cap timeout 900 $TR --nproc-per-node 4 --master-port 2965$i bench.py --gpus 4 --exposed --no-cpu-baseline > $O/gpt_cap$cap.json 2>$O/gpt_cap$cap.err
done
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), (d.get('exposed_comm') or {}).get('frac_of_step'), d['clocks']['sm_mhz'], {k:(round(v['mean_ms'],3)) for k,v in d['kernels'].items()})" || tail -5 ${f%.json}.err; done
