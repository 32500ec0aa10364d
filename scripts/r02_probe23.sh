#!/bin/bash
# e2e with the loss readback (and the dx-readback variant) at N = 1 and 4
O=gpurun_out/r02aa; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
B="bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
timeout 400 python $B > $O/mixtral_n1.log 2>&1
timeout 400 $TR --nproc-per-node=4 --master-port=29851 $B --gpus 4 > $O/mixtral_n4.log 2>&1
timeout 400 python $B --no-graph > $O/mixtral_n1_nograph.log 2>&1
echo done
