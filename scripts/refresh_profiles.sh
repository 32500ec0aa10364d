#!/bin/bash
# Regenerates the round's bench lines, traces and ncu evidence on a 4-GPU box:
#   /usr/local/graft/bin/gpurun --gpus 4 --timeout 2700 -- scripts/refresh_profiles.sh
# Outputs land in gpurun_out/prof/ (copied into profiles/ by hand after review).
O=gpurun_out/prof
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1"
run() { local name=$1; shift; echo "== $name"; timeout 420 "$@" > $O/$name.log 2>&1; echo "rc=$?"; tail -1 $O/$name.log | cut -c1-160; }
run bench_mixtral_n1 python bench.py --trace $O/trace_mixtral_n1.json
run bench_reference_n1 python bench.py --impl reference
run bench_mixtral_n2 $TR --nproc-per-node=2 --master-port=29601 bench.py --gpus 2 --trace $O/trace_mixtral_n2.json
run bench_mixtral_n4 $TR --nproc-per-node=4 --master-port=29602 bench.py --gpus 4 --trace $O/trace_mixtral_n4.json
run bench_reference_n4 $TR --nproc-per-node=4 --master-port=29603 bench.py --gpus 4 --impl reference
run bench_deepseek_n4 $TR --nproc-per-node=4 --master-port=29604 bench.py --gpus 4 --config deepseek
run bench_fp8zipf_n4 $TR --nproc-per-node=4 --master-port=29605 bench.py --gpus 4 --config mixtral_fp8_zipf
run bench_attn_n4 $TR --nproc-per-node=4 --master-port=29606 bench.py --gpus 4 --config attn
run bench_ulysses_n4 $TR --nproc-per-node=4 --master-port=29607 bench.py --gpus 4 --config ulysses
run bench_dp_n4 $TR --nproc-per-node=4 --master-port=29608 bench.py --gpus 4 --config dp
run bench_deepseek_n1 python bench.py --config deepseek --no-nccl-baseline
run bench_small_n1 python bench.py --config small --no-nccl-baseline
# launch list of one eager step (cold-cache, serialised: shares, not absolutes)
echo "== ncu launches"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mixtral_n1.csv \
    python scripts/profile_step.py > $O/ncu_launches.log 2>&1; echo "rc=$?"
# full capture of the six GEMMs of the second step
echo "== ncu full"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm -s 6 -c 6 \
    -o $O/gemms_mixtral_n1 python scripts/profile_step.py > $O/ncu_full.log 2>&1; echo "rc=$?"
ncu -i $O/gemms_mixtral_n1.ncu-rep --page raw --csv > $O/gemms_ncu_raw.csv 2>/dev/null
echo done
