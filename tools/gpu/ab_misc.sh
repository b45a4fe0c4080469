O=gpurun_out/misc; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 900 $TR --nproc-per-node 4 --master-port 2962$i bench.py --gpus 4 --opt-in-bwd --no-cpu-baseline > $O/bench_n4_optbwd_$i.json 2>/dev/null
timeout 900 $TR --nproc-per-node 4 --master-port 2963$i bench.py --gpus 4 --no-cpu-baseline > $O/bench_n4_default_$i.json 2>/dev/null
done
FSDP_ADAM_VARIANT=3 timeout 600 python bench.py --steps 8 --no-cpu-baseline > $O/bench_n1_adamv3.json 2>/dev/null
FSDP_ADAM_VARIANT=0 timeout 600 python bench.py --steps 8 --no-cpu-baseline > $O/bench_n1_adamv0.json 2>/dev/null
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), d['roofline']['mean_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
