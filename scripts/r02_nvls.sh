#!/bin/bash
mkdir -p gpurun_out/r02n
timeout 120 ./scripts/probe_nvls.bin > gpurun_out/r02n/probe.log 2>&1; echo "rc=$?" >> gpurun_out/r02n/probe.log
nvidia-smi -q | grep -i -A3 "fabric\|nvlink" | head -40 >> gpurun_out/r02n/smi.log 2>&1
echo done
