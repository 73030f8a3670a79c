#!/bin/bash
# A/B of the row-copy minimum row bytes (TT_KNOB_ROW_MIN, default 512)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/rowmin
for th in 1024 2048 4096; do
  timeout 900 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 3 --reps 7 --env TT_KNOB_ROW_MIN=$th \
    > gpurun_out/rowmin/ab_$th.txt 2>&1
done
