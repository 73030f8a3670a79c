#!/bin/bash
# A/B of the 2-D kernel's output-side fill threshold (TT_KNOB_T2D_FILLB):
# only cases whose plan changes are timed (tools/ab_opts.py --env)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/fillb
for th in 0.8 0.9; do
  timeout 900 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 3 --reps 7 --env TT_KNOB_T2D_FILLB=$th \
    > gpurun_out/fillb/ab_$th.txt 2>&1
done
