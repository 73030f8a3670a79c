#!/bin/bash
# A/B of balanced split chunks in the generic tile (TT_KNOB_SPLIT_BAL)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/bal
for th in 0.8 0.9; do
  timeout 1200 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 3 --reps 5 --env TT_KNOB_SPLIT_BAL=$th \
    > gpurun_out/bal/ab_$th.txt 2>&1
done
