#!/bin/bash
O=gpurun_out/r02y
mkdir -p $O
timeout 400 python bench.py --no-cpu-baseline --no-integer-compare --no-gemm-compare > $O/bench_n1.log 2>&1
timeout 600 python -m pytest tests/test_gpu_routing.py tests/test_gpu_quant.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
echo done
