#!/bin/bash
# tail-tile cost + torch._grouped_mm kernel identity at the fc1 / fc2-dgrad shapes
mkdir -p gpurun_out/r02i
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/r02i/smi.txt
timeout 300 python scripts/gemm_tail_probe.py > gpurun_out/r02i/probe.json 2> gpurun_out/r02i/probe.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,launch__registers_per_thread \
  --clock-control none --csv --log-file gpurun_out/r02i/ncu.csv python scripts/gemm_tail_probe.py --ncu > gpurun_out/r02i/ncu.log 2>&1
echo done
