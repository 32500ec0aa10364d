#!/bin/bash
# Same-box A/B against a built worktree of another commit (git worktree add ab/<name> <commit>;
# make -C ab/<name> paper_2505_11432_b200/libmoe_b200.so), selected with AB_BASE=<name>.
# usage: ab/run_ab_phase.sh <reps> <script relative to repo root>
reps=$1; script=$2
for i in $(seq $reps); do
  for v in base new; do
    if [ $v = base ]; then d=ab/${AB_BASE:-base}; else d=.; fi
    (cd $d && echo "$v $(python /root/repo/$script 2>&1 | tail -1)")
  done
done
