O=gpurun_out/split; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -2 $O/pytest_mgpu.log
i=0
for sp in 2 0 2 0; do
i=$((i+1))
timeout 900 $TR --nproc-per-node 4 --master-port 2966$i bench.py --gpus 4 --opt-split-first $sp --no-cpu-baseline > $O/gpt_s${sp}_$i.json 2>$O/gpt_$i.err
done
for sp in 2 0; do
i=$((i+1))
timeout 1200 $TR --nproc-per-node 4 --master-port 2966$i bench.py --gpus 4 --config t5-11b --steps 6 --opt-split-first $sp --no-cpu-baseline > $O/t5_s${sp}.json 2>$O/t5_$i.err
done
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/d['n_gpus'],1), d['clocks']['sm_mhz'], json.dumps(d.get('comm_stalls_top_units',{}).get('allgather', [])[:3]))" || tail -3 $O/*.err; done
