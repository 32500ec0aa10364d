#!/bin/bash
O=gpurun_out/r02ag; mkdir -p $O
timeout 600 python scripts/probe_fused_n1.py > $O/fused_n1.json 2> $O/fused_n1.err
echo done
