#!/bin/bash
# AG-GEMM: partial last wave as M = 128 pair tiles (split_last) vs full tiles
O=gpurun_out/r02ae; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_attn.py -v -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  timeout 300 $TR --master-port=2995$i bench.py --gpus 4 --config attn > $O/split_$i.log 2>&1
  MOE_ATTN_NO_TAIL_SPLIT=1 timeout 300 $TR --master-port=2996$i bench.py --gpus 4 --config attn > $O/nosplit_$i.log 2>&1
done
echo done
