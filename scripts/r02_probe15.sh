#!/bin/bash
# fused GEMM-RS with a signal warp (epilogue warps never fence), TP = 4
O=gpurun_out/r02ab; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_attn.py -v -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  for d in 6; do
    MOE_ATTN_RS_DELAY=$d timeout 300 $TR --master-port=2979$i bench.py --gpus 4 --config attn > $O/fused_d${d}_$i.log 2>&1
  done

  MOE_ATTN_RS_UNFUSED=1 timeout 300 $TR --master-port=2977$i bench.py --gpus 4 --config attn > $O/unfused_$i.log 2>&1
done
echo done
