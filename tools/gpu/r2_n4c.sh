#!/bin/bash
# fused-cast all-gather A/B, T5-11B on the round-2 code, CE reduce-scatter
# pipelining at unit sizes, and the N=1 ncu evidence (launch list + Adam capture).
O=gpurun_out/${OUT:-r2n4c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --exposed > $O/bench_n4.json 2> $O/bench_n4.err
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --exposed --fused-cast-ag > $O/bench_n4_fused_cast.json 2> $O/bench_n4_fused_cast.err
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --exposed --fused-cast-ag --ag-engine nvls > $O/bench_n4_fused_cast_nvls.json 2> $O/bench_n4_fused_cast_nvls.err
timeout 1500 python bench.py --gpus 4 --config t5-11b --steps 6 --warmup 3 --exposed > $O/bench_t5_11b_n4.json 2> $O/bench_t5_11b_n4.err
RS_SIZES_MB=100,256,537 RS_VARIANTS=pull_p1,push_geo_u8M,push_geo_u4M,pull_uni_u8M \
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29541 tools/rs_ce_sweep.py > $O/rs_ce_n4.json 2> $O/rs_ce_n4.err
# N=1 evidence on GPU 0: clean bench, then the ncu launch list of the same command, then one full capture of Adam
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_n1.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:adam_tma --launch-count 1 \
  -o $O/ncu_adam_n1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_adam.log 2>&1
echo done
