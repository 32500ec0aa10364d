#!/bin/bash
# e2e vs value at N = 4: host-copy floor
O=gpurun_out/r02v; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
B="bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
timeout 400 $TR --nproc-per-node=4 --master-port=29811 $B --gpus 4 > $O/mixtral_n4.log 2>&1
timeout 400 $TR --nproc-per-node=2 --master-port=29812 $B --gpus 2 > $O/mixtral_n2.log 2>&1
echo done
