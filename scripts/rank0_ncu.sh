#!/bin/bash
# torchrun --no-python entry: rank 0 runs under ncu with a single-pass metric
# set (no kernel replay, so the peers' flag waits are never stalled by replays);
# the other ranks run plain. NCU_OUT / NCU_METRICS / NCU_KERNELS from the env.
if [ "$RANK" = "0" ]; then
  exec ncu --metrics "${NCU_METRICS}" --clock-control none -k "regex:${NCU_KERNELS:-grouped_gemm}" \
       --csv --log-file "${NCU_OUT}" python "$@"
else
  exec python "$@"
fi
