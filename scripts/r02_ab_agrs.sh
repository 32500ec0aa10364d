#!/bin/bash
# Same-box A/B of the round-1 build (ab/base) vs the working tree at N=4 (Mixtral),
# the ag_rs pattern tests, and DeepSeek N=4 with both EP patterns.
O=gpurun_out/r02
mkdir -p $O
AB_BASE=base bash scripts/ab_ab4.sh 2 4 > $O/ab_n4_mixtral.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -v -rs -s -k "ag_rs" > $O/pytest_agrs.log 2>&1; echo "rc=$?" >> $O/pytest_agrs.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node=4"
for p in a2a ag_rs; do
  timeout 500 $TR --master-port=29621 bench.py --gpus 4 --config deepseek --no-nccl-baseline --no-cpu-baseline --ep-pattern $p > $O/bench_deepseek_n4_$p.log 2>&1
  echo "$p rc=$?" >> $O/bench_deepseek_n4_$p.log
  timeout 500 $TR --master-port=29631 bench.py --gpus 4 --config mixtral --no-nccl-baseline --no-cpu-baseline --ep-pattern $p > $O/bench_mixtral_n4_$p.log 2>&1
  echo "$p rc=$?" >> $O/bench_mixtral_n4_$p.log
done
echo done
