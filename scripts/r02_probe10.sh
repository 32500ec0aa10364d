#!/bin/bash
mkdir -p gpurun_out/r02j
timeout 300 python scripts/gemm_power_probe.py > gpurun_out/r02j/power.json 2> gpurun_out/r02j/power.err
echo done
