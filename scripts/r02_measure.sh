#!/bin/bash
# N=1 bench (cpu_baseline, integer path, gemm_vs_cublas, graph trace), N=4 bench +
# trace, NVLink byte counters of the fused GEMMs at EP=4 (rank 0 under ncu, one pass).
O=gpurun_out/r02m
mkdir -p $O
timeout 900 python bench.py --trace $O/trace_mixtral_n1.json > $O/bench_n1.log 2>&1; echo "rc=$?" >> $O/bench_n1.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node=4"
timeout 600 $TR --master-port=29651 bench.py --gpus 4 --trace $O/trace_mixtral_n4.json > $O/bench_n4.log 2>&1; echo "rc=$?" >> $O/bench_n4.log
M="gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for cfg in mixtral deepseek; do
  for p in a2a ag_rs; do
    NCU_OUT=$O/nvlink_${cfg}_${p}_n4.csv NCU_METRICS=$M MOE_EP_PATTERN=$p STEPS=2 timeout 600 \
      $TR --master-port=29652 --no-python scripts/rank0_ncu.sh scripts/profile_step_ep.py $cfg > $O/nvlink_${cfg}_${p}.log 2>&1
    echo "$cfg $p rc=$?" >> $O/nvlink_${cfg}_${p}.log
  done
done
echo done
