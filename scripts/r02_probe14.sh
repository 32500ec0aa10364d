#!/bin/bash
# fused GEMM-RS cost split (timing probes; diag runs give wrong y by design)
O=gpurun_out/r02n; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
for i in 1 2; do
  for dg in 0 1 2 3; do
    MOE_ATTN_RS_DIAG=$dg MOE_ATTN_RS_DELAY=6 timeout 300 $TR --master-port=2979$i bench.py --gpus 4 --config attn > $O/fused_diag${dg}_$i.log 2>&1
  done
  MOE_ATTN_RS_UNFUSED=1 timeout 300 $TR --master-port=2977$i bench.py --gpus 4 --config attn > $O/unfused_$i.log 2>&1
done
echo done
