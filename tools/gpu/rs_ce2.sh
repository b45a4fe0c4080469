RS_VARIANTS=push_p4,push_p4_r32,push_p4_r64,pull_p4_r32,push_p8_r32,push_p16_r16 RS_SIZES_MB=256,1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 tools/rs_ce_sweep.py > gpurun_out/rs_ce2_n4.json 2> gpurun_out/rs_ce2_n4.err
grep -v OMP gpurun_out/rs_ce2_n4.err | grep -v "\*\*\*" | tail -12
