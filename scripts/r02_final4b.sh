#!/bin/bash
# Refresh of the round-2 4-GPU evidence after the fp32 / baseline / trace changes.
O=gpurun_out/r02g
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -v -rs -s > $O/pytest_gpu_n4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_n4.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log; }
run bench_mixtral_n1 python bench.py --trace $O/trace_mixtral_n1.json
run bench_mixtral_n4 $TR --nproc-per-node=4 --master-port=29721 bench.py --gpus 4 --trace $O/trace_mixtral_n4.json
run bench_mixtral_n2 $TR --nproc-per-node=2 --master-port=29722 bench.py --gpus 2 --trace $O/trace_mixtral_n2.json
run bench_deepseek_n4 $TR --nproc-per-node=4 --master-port=29723 bench.py --gpus 4 --config deepseek --trace $O/trace_deepseek_n4.json
run bench_attn_n4 $TR --nproc-per-node=4 --master-port=29724 bench.py --gpus 4 --config attn
run bench_small_f32 python bench.py --config small_f32
run bench_deepseek_n1 python bench.py --config deepseek --no-nccl-baseline --no-cpu-baseline --no-integer-compare
echo done
