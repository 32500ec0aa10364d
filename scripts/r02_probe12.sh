#!/bin/bash
# GEMM-RS variants at TP = 4: fused (lane-0 release only / every lane fences), unfused (interleaved / shard chunks)
O=gpurun_out/r02l; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_attn.py -v -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  timeout 300 $TR --master-port=2975$i bench.py --gpus 4 --config attn > $O/fused_rel_$i.log 2>&1
  MOE_ATTN_RS_FENCE_ALL=1 timeout 300 $TR --master-port=2976$i bench.py --gpus 4 --config attn > $O/fused_fenceall_$i.log 2>&1
  MOE_ATTN_RS_UNFUSED=1 timeout 300 $TR --master-port=2977$i bench.py --gpus 4 --config attn > $O/unfused_$i.log 2>&1
  MOE_ATTN_RS_UNFUSED=1 MOE_ATTN_RS_CHUNK=1 timeout 300 $TR --master-port=2978$i bench.py --gpus 4 --config attn > $O/unfused_chunk_$i.log 2>&1
done
echo done
