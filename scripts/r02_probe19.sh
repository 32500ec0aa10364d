#!/bin/bash
# RematPolicy::off (no fc2_in recompute in the fc2-dgrad epilogue): bit-exactness and step time;
# e2e host-copy floor field
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-cpu-baseline --no-nccl-baseline --no-integer-compare --no-gemm-compare"
for i in 1 2; do
  timeout 300 $B > $O/mixtral_remat_$i.log 2>&1
  timeout 300 $B --no-remat > $O/mixtral_noremat_$i.log 2>&1
done
echo done
