#!/bin/bash
O=gpurun_out/r02e
mkdir -p $O
timeout 400 python bench.py --no-cpu-baseline --no-integer-compare --no-gemm-compare --no-nccl-baseline > $O/bench_n1.log 2>&1
timeout 500 python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node=2 --master-port=29731 bench.py --gpus 2 --no-nccl-baseline > $O/bench_n2.log 2>&1
echo done
