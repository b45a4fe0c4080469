set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ll4.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_ll4.log
FSDP_SWEEP_SIZES=0.25,1,2,4,8,16,64 FSDP_SWEEP_CTAS=16,32,64 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 bench.py --mode sweep > gpurun_out/sweep_ll_n4.json 2> gpurun_out/sweep_ll_n4.err
tail -3 gpurun_out/sweep_ll_n4.err
