#!/bin/bash
# Round-2 final 1-GPU evidence: N = 1 bench lines, the reference CPU arm, the
# launch list and a full ncu capture of the six GEMMs. Outputs in gpurun_out/r02x/.
O=gpurun_out/r02x
mkdir -p $O
run() { local name=$1; shift; timeout 600 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log; }
run bench_mixtral_n1 python bench.py --trace $O/trace_mixtral_n1.json
run bench_reference_n1 python bench.py --impl reference --steps 5
run bench_small_f32 python bench.py --config small_f32
run bench_deepseek_n1 python bench.py --config deepseek --no-nccl-baseline --no-cpu-baseline --no-integer-compare
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mixtral_n1.csv \
    python scripts/profile_step.py > $O/ncu_launches.log 2>&1; echo "rc=$?" >> $O/ncu_launches.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm -s 6 -c 6 \
    -o $O/gemms_mixtral_n1 python scripts/profile_step.py > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
ncu -i $O/gemms_mixtral_n1.ncu-rep --page raw --csv > $O/gemms_ncu_raw.csv 2>/dev/null
echo done
