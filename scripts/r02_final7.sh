#!/bin/bash
# The driver's round-end configuration on the final build: smoke() and pytest -m gpu on one GPU.
O=gpurun_out/r02af; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu_n1.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_n1.log
echo done
