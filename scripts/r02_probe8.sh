#!/bin/bash
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -k "timeout or protocol" -v -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
echo done
