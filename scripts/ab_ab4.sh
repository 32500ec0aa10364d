#!/bin/bash
# Same-box A/B against a built worktree of another commit (git worktree add ab/<name> <commit>;
# make -C ab/<name> paper_2505_11432_b200/libmoe_b200.so), selected with AB_BASE=<name>.
# usage: ab/run_ab4.sh <reps> <ngpu> <bench args...>
reps=$1; n=$2; shift; shift
for i in $(seq $reps); do
  for v in base new nodedup; do
    d=.; unset MOE_NO_DISPATCH_DEDUP
    if [ $v = base ]; then d=ab/${AB_BASE:-base}; fi
    if [ $v = nodedup ]; then export MOE_NO_DISPATCH_DEDUP=1; fi
    (cd $d && timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=29694 bench.py --gpus $n --no-nccl-baseline --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['exposed_comm']['exposed_pct'],1))")
  done
done
