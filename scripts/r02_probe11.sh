#!/bin/bash
# fused GEMM-RS (reduce in the own-shard epilogue) vs staging + barrier + reduce, TP = 4
O=gpurun_out/r02k; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_attn.py -v -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  timeout 300 $TR --master-port=2973$i bench.py --gpus 4 --config attn > $O/attn_fused_$i.log 2>&1
  MOE_ATTN_RS_UNFUSED=1 timeout 300 $TR --master-port=2974$i bench.py --gpus 4 --config attn > $O/attn_unfused_$i.log 2>&1
done
echo done
