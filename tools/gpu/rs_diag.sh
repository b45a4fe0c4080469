MP_ONLY=deadlock_detection timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29510 tests/mp_worker.py 2>&1 | grep -E "world|Error" | head -5
RS_VARIANTS=ag_ce,push_p1,push_p1_noreduce,pull_p1,pull_p1_noreduce,push_geo_4M,push_geo_noreduce RS_SIZES_MB=256,1024,2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 tools/rs_ce_sweep.py > gpurun_out/rs_diag_n4.json 2> gpurun_out/rs_diag_n4.err
grep -v OMP gpurun_out/rs_diag_n4.err | grep -v "\*\*\*" | tail -12
