set -x
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_collectives.py -x -q -k "ll" 2>&1 | tail -15
MP_ONLY=ll_collectives timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 tests/mp_worker.py 2>&1 | tail -20
FSDP_SWEEP_SIZES=0.25,1,4,16,64 FSDP_SWEEP_CTAS=16,32 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --mode sweep > gpurun_out/sweep_ll_n2.json 2> gpurun_out/sweep_ll_n2.err
tail -3 gpurun_out/sweep_ll_n2.err
