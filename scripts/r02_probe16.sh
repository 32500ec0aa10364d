#!/bin/bash
# tails-last tile order for the long-K GEMMs (fc1 dgrad, fc2): parity, step time, ncu DRAM
O=gpurun_out/r02q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_gemm.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_fullshape.py -q -x -k "mixtral or deepseek" > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
B="python bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
for i in 1 2; do
  for tl in 0 1 3; do
    MOE_TAILS_LAST=$tl timeout 300 $B > $O/mixtral_tl${tl}_$i.log 2>&1
  done
done
for tl in 0 1; do
  MOE_TAILS_LAST=$tl timeout 300 $B --config deepseek > $O/deepseek_tl${tl}.log 2>&1
done
for tl in 0 1 3; do
  MOE_TAILS_LAST=$tl STEPS=2 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:grouped_gemm \
    --clock-control none --csv --log-file $O/ncu_tl$tl.csv python scripts/profile_step.py > $O/ncu_tl$tl.log 2>&1
done
echo done
