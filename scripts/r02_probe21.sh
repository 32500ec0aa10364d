#!/bin/bash
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "cf1" -v -s > $O/pytest_cf1.log 2>&1; echo "rc=$?" >> $O/pytest_cf1.log
echo done
