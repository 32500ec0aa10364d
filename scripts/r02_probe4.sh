#!/bin/bash
O=gpurun_out/r02x
mkdir -p $O
timeout 300 python scripts/probe_f32.py err > $O/err_bf16x6.log 2>&1
timeout 300 python scripts/probe_accum.py > $O/accum.log 2>&1
timeout 900 python -m pytest tests/test_gpu_f32.py -q -x -s > $O/pytest_f32.log 2>&1; echo "rc=$?" >> $O/pytest_f32.log
timeout 300 python bench.py --config small_f32 > $O/bench_small_f32.log 2>&1
MOE_F32_FFMA=1 timeout 300 python bench.py --config small_f32 > $O/bench_small_f32_ffma.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bf16x6.csv python scripts/probe_f32.py > $O/ncu.log 2>&1
echo done
