run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 --steps 10 --warmup 3 --exposed --no-cpu-baseline 2>/dev/null | tail -1; }
MP_ONLY=ce_schedules timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29510 tests/mp_worker.py 2>&1 | grep world
for i in 1 2; do
FSDP_CE_RS_PUSH=0 run 2951$i > gpurun_out/ab_pull_$i.json
FSDP_CE_RS_PUSH=1 run 2952$i > gpurun_out/ab_push_$i.json
done
for f in gpurun_out/ab_pu*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value']/d['n_gpus'], d.get('exposed_comm',{}).get('frac'), d.get('comm_stalls',{}).get('reduce_scatter_end'))"; done
