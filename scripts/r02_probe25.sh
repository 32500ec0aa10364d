#!/bin/bash
O=gpurun_out/r02ad; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_quant.py tests/test_gpu_layer.py tests/test_gpu_gemm.py -q -x > $O/pytest_1.log 2>&1; echo "rc=$?" >> $O/pytest_1.log
timeout 900 python -m pytest tests/test_gpu_fullshape.py -k fp8 -q -x -s > $O/pytest_2.log 2>&1; echo "rc=$?" >> $O/pytest_2.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -k "fp8 or protocol or ep2" -q -x -s > $O/pytest_3.log 2>&1; echo "rc=$?" >> $O/pytest_3.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
timeout 300 $TR --nproc-per-node=4 --master-port=29891 bench.py --gpus 4 --config mixtral_fp8_zipf --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare > $O/fp8zipf_n4.log 2>&1
echo done
