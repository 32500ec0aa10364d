#!/bin/bash
O=gpurun_out/r02r; mkdir -p $O
for v in mn8 km8 mn1 mn8s; do
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    -k regex:grouped_gemm --clock-control none --csv --log-file $O/ncu_$v.csv python scripts/probe_fc1d_dram.py $v > $O/ncu_$v.log 2>&1
  MOE_STATIC_TILES=1 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:grouped_gemm --clock-control none --csv --log-file $O/ncu_${v}_static.csv python scripts/probe_fc1d_dram.py $v > $O/ncu_${v}_static.log 2>&1
done
echo done
