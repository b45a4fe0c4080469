RS_VARIANTS=push_geo_p3,push_geo_p4,push_geo_p5,push_geo_4M RS_SIZES_MB=256,1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 tools/rs_ce_sweep.py > gpurun_out/rs_diag3_n4.json 2> gpurun_out/rs_diag3_n4.err
grep -v OMP gpurun_out/rs_diag3_n4.err | grep -v "\*\*\*" | tail -12
