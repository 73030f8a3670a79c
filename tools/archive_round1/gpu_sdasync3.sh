#!/bin/bash
# fp64 generic-tile cases: slot-dim map with a cp.async ring (options) vs the heuristic plan
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/sdasync3
O=gpurun_out/sdasync3
for S in 3 4; do
  timeout 1200 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 1 --reps 5 --esize 8 --kernel-filter tile slot_dims=1 stages=$S > $O/ab8_$S.txt 2>&1
done
