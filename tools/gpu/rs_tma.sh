V=$(python -c "print(','.join(f'tma_r{r}_c{c}' for r in range(4) for c in (64,128)))")
RS_VARIANTS=$V RS_SIZES_MB=256,1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 tools/rs_ce_sweep.py > gpurun_out/rs_tma_n4.json 2> gpurun_out/rs_tma_n4.err
grep -v OMP gpurun_out/rs_tma_n4.err | grep -v "\*\*\*" | tail -10
V=$(python -c "print(','.join(f'tma_r{r}_c128' for r in range(4)))")
RS_VARIANTS=$V RS_SIZES_MB=1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29513 tools/rs_ce_sweep.py > gpurun_out/rs_tma_n2.json 2> gpurun_out/rs_tma_n2.err
grep -v OMP gpurun_out/rs_tma_n2.err | grep -v "\*\*\*" | tail -10
