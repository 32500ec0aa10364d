#!/bin/bash
# fused GEMM-RS own-tile delay D with whole-line stores, TP = 4
O=gpurun_out/r02ai; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for d in 3 6 12; do
  MOE_ATTN_RS_DELAY=$d timeout 200 $TR --master-port=2997$d bench.py --gpus 4 --config attn > $O/d$d.log 2>&1
done
echo done
