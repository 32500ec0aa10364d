#!/bin/bash
# Final multi-GPU check of the last build: the n > 1 GPU tests and the key N = 2 / 4 bench lines.
O=gpurun_out/r02w2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_attn.py tests/test_gpu_ulysses.py tests/test_gpu_dp.py -v -rs > $O/pytest_multi_n4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_multi_n4.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log; }
run bench_mixtral_n4 $TR --nproc-per-node=4 --master-port=29931 bench.py --gpus 4 --trace $O/trace_mixtral_n4.json
run bench_mixtral_n2 $TR --nproc-per-node=2 --master-port=29932 bench.py --gpus 2 --trace $O/trace_mixtral_n2.json
run bench_deepseek_n4 $TR --nproc-per-node=4 --master-port=29933 bench.py --gpus 4 --config deepseek --trace $O/trace_deepseek_n4.json
run bench_attn_n4 $TR --nproc-per-node=4 --master-port=29936 bench.py --gpus 4 --config attn
run bench_ulysses_n4 $TR --nproc-per-node=4 --master-port=29937 bench.py --gpus 4 --config ulysses
echo done
