#!/bin/bash
# Round-2 GPU check: full pytest -m gpu (n>1 cases included on a 4-GPU box),
# then N=1 and N=4 Mixtral bench lines. Outputs in gpurun_out/r02/.
O=gpurun_out/r02
mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt; lscpu | head -20 >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -v -rs -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > $O/bench_n1.log 2>&1; echo "rc=$?" >> $O/bench_n1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29611 \
    bench.py --gpus 4 --no-cpu-baseline > $O/bench_n4.log 2>&1; echo "rc=$?" >> $O/bench_n4.log
echo done
