#!/bin/bash
O=gpurun_out/r02q
mkdir -p $O
timeout 300 python scripts/nvml_nvlink_probe.py > $O/nvml_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attn.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node=2"
for bn in 256 128; do
  MOE_ATTN_QKV_BN=$bn timeout 300 $TR --master-port=29712 bench.py --gpus 2 --config attn > $O/attn_n2_bn$bn.log 2>&1
done
echo done
