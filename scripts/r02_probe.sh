#!/bin/bash
# Tests of the new operators, N=1 A/B probes (fused vs unfused dispatch, router
# split), the fp32 configs[0] line, a full ncu capture of the six GEMMs and the
# compute-sanitizer runs. Outputs in gpurun_out/r02p/.
O=gpurun_out/r02p
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullshape.py tests/test_gpu_quant.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-cpu-baseline --no-gemm-compare --no-integer-compare"
for i in 1 2; do
  timeout 300 $B > $O/bench_default_$i.log 2>&1
  MOE_UNFUSED_DISPATCH=1 timeout 300 $B > $O/bench_unfused_$i.log 2>&1
  MOE_ROUTER_SPLIT=1 timeout 300 $B > $O/bench_split1_$i.log 2>&1
  timeout 300 $B --no-graph > $O/bench_nograph_$i.log 2>&1
done
timeout 300 python bench.py --config small_f32 > $O/bench_small_f32.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm -s 6 -c 6 \
    -o $O/gemms_mixtral_n1 python scripts/profile_step.py > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mixtral_n1.csv \
    python scripts/profile_step.py > $O/ncu_launches.log 2>&1
bash scripts/sanitize.sh
mv gpurun_out/sanitize $O/ 2>/dev/null
echo done
