#!/bin/bash
# compute-sanitizer runs of the layer's kernels (memcheck incl. the cross-GPU
# flag / peer-pointer protocol at EP=2, racecheck + synccheck on shared memory
# and barriers, initcheck on global reads). Logs in gpurun_out/sanitize/.
O=gpurun_out/sanitize
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 python scripts/sanitize_layer.py > $O/${tool}_n1.log 2>&1
  echo "rc=$?" >> $O/${tool}_n1.log
done
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --nproc-per-node=2 --master-port=29671 \
  --no-python $CS --tool memcheck --print-limit 50 python scripts/sanitize_layer.py > $O/memcheck_n2.log 2>&1
echo "rc=$?" >> $O/memcheck_n2.log
fi
echo done
