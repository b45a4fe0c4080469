timeout 600 python tools/adam_bench.py > gpurun_out/adam_variants4.json 2> gpurun_out/adam_variants4.err; cut -c1-20,100-300 gpurun_out/adam_variants4.err
for v in 0 1 2 3 4; do
FSDP_ADAM_VARIANT=$v timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/adam_instep_v$v.json
python -c "
import json; d=json.load(open('gpurun_out/adam_instep_v$v.json')); print('v$v', d['value'], d['roofline']['mean_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
