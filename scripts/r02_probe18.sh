#!/bin/bash
# bulk-copy router kernel vs the register-streaming one (Mixtral shape): parity, ncu time, step
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_routing.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_fullshape.py -q -x -k "mixtral" > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
for rk in bulk regs; do
  MOE_ROUTER_KERNEL=$rk STEPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    -k regex:router_logits --clock-control none --csv --log-file $O/ncu_$rk.csv python scripts/profile_step.py > $O/ncu_$rk.log 2>&1
done
B="python bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
for i in 1 2; do
  for rk in bulk regs; do
    MOE_ROUTER_KERNEL=$rk timeout 300 $B > $O/mixtral_${rk}_$i.log 2>&1
  done
done
echo done
