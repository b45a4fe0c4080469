#!/bin/bash
# end-of-round AG/RS sweep vs NCCL at W = 4 and W = 2, and the layout kernels vs the HBM roofline
O=gpurun_out/${OUT:-r2sweepfinal}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
FSDP_SWEEP_SIZES=1,16,64,128,256,1024,2048 timeout 1500 python bench.py --gpus 4 --mode sweep > $O/sweep_n4.json 2> $O/sweep_n4.err
echo "sweep4 rc=$?" >> $O/times.txt
FSDP_SWEEP_SIZES=1,16,64,256,2048 timeout 1500 python bench.py --gpus 2 --mode sweep > $O/sweep_n2.json 2> $O/sweep_n2.err
echo "sweep2 rc=$?" >> $O/times.txt
timeout 900 python bench.py --mode copy > $O/copy_n1.json 2> $O/copy_n1.err
echo "copy rc=$?" >> $O/times.txt
