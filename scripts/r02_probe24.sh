#!/bin/bash
# 128-byte row segments in the store / scatter epilogues vs 64-byte (MOE_EPI_STORE32=1), same box
O=gpurun_out/r02ac; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
B="bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py tests/test_gpu_ulysses.py tests/test_gpu_attn.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  for v in 0 1; do
    if [ $v = 1 ]; then export MOE_EPI_STORE32=1; else unset MOE_EPI_STORE32; fi
    timeout 300 $TR --nproc-per-node=4 --master-port=2986$i $B --gpus 4 --config deepseek > $O/deepseek_s32_${v}_$i.log 2>&1
    timeout 300 $TR --nproc-per-node=4 --master-port=2987$i $B --gpus 4 > $O/mixtral_s32_${v}_$i.log 2>&1
    timeout 300 $TR --nproc-per-node=4 --master-port=2988$i bench.py --gpus 4 --config ulysses > $O/ulysses_s32_${v}_$i.log 2>&1
  done
done
unset MOE_EPI_STORE32
echo done
