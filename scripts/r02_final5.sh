#!/bin/bash
# Round-2 final 4-GPU evidence: the whole GPU test suite (n = 1, 2, 4 cases) and
# the multi-GPU bench lines with traces. Outputs in gpurun_out/r02w/.
O=gpurun_out/r02w
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -v -rs > $O/pytest_gpu_n4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_n4.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log; }
run bench_mixtral_n4 $TR --nproc-per-node=4 --master-port=29831 bench.py --gpus 4 --trace $O/trace_mixtral_n4.json
run bench_mixtral_n2 $TR --nproc-per-node=2 --master-port=29832 bench.py --gpus 2 --trace $O/trace_mixtral_n2.json
run bench_deepseek_n4 $TR --nproc-per-node=4 --master-port=29833 bench.py --gpus 4 --config deepseek --trace $O/trace_deepseek_n4.json
run bench_deepseek_n4_ag_rs $TR --nproc-per-node=4 --master-port=29834 bench.py --gpus 4 --config deepseek --ep-pattern ag_rs --no-nccl-baseline
run bench_fp8zipf_n4 $TR --nproc-per-node=4 --master-port=29835 bench.py --gpus 4 --config mixtral_fp8_zipf
run bench_attn_n4 $TR --nproc-per-node=4 --master-port=29836 bench.py --gpus 4 --config attn
run bench_ulysses_n4 $TR --nproc-per-node=4 --master-port=29837 bench.py --gpus 4 --config ulysses
run bench_dp_n4 $TR --nproc-per-node=4 --master-port=29838 bench.py --gpus 4 --config dp
echo done
