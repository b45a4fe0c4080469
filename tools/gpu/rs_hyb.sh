MP_ONLY=ce_schedules timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29510 tests/mp_worker.py 2>&1 | grep -E "world|Error|rror" | head -5
RS_VARIANTS=push_geo_4M,hyb_f10,hyb_f20,hyb_f30,hyb_f40 RS_SIZES_MB=256,1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 tools/rs_ce_sweep.py > gpurun_out/rs_hyb_n4.json 2> gpurun_out/rs_hyb_n4.err
grep -v OMP gpurun_out/rs_hyb_n4.err | grep -v "\*\*\*" | tail -8
