#!/bin/bash
# Same-box A/B against a built worktree of another commit (git worktree add ab/<name> <commit>;
# make -C ab/<name> paper_2505_11432_b200/libmoe_b200.so), selected with AB_BASE=<name>.
# usage: ab/run_ab.sh <reps> <bench args...>: alternates ab/base and the working tree
reps=$1; shift
for i in $(seq $reps); do
  for v in base new; do
    if [ $v = base ]; then d=ab/${AB_BASE:-base}; else d=.; fi
    (cd $d && timeout 300 python bench.py --no-nccl-baseline --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']
print('$v', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['gpu_launches'], 'e2e', round(d['e2e']['value']), 'fc2dg', round(p['fc2_dgrad'],3), 'sum', round(sum(p.values()),3))")
  done
done
