#!/bin/bash
O=gpurun_out/r02t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_gemm.py -q -x -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config small_f32 > $O/bench_small_f32_tf32.log 2>&1
MOE_F32_FFMA=1 timeout 300 python bench.py --config small_f32 > $O/bench_small_f32_ffma.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-integer-compare > $O/bench_mixtral_n1.log 2>&1
echo done
