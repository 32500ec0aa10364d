#!/bin/bash
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullshape.py -k fp8 -v -s > $O/pytest_fp8_n1.log 2>&1; echo "rc=$?" >> $O/pytest_fp8_n1.log
timeout 900 python -m pytest tests/test_gpu_multi.py -k "fp8" -v -s > $O/pytest_fp8_n4.log 2>&1; echo "rc=$?" >> $O/pytest_fp8_n4.log
echo done
