#!/bin/bash
# after restoring 32-column local epilogue stores: GEMM / layer tests, then the 1-GPU evidence
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_fullshape.py -q -x > $O/pytest_n1.log 2>&1; echo "rc=$?" >> $O/pytest_n1.log
bash scripts/r02_final5b.sh
