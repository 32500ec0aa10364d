#!/bin/bash
O=gpurun_out/r02ah; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attn.py -v -s > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
echo done
