#!/bin/bash
O=gpurun_out/r02v
mkdir -p $O
timeout 300 python scripts/probe_accum.py > $O/accum.log 2>&1
echo done
