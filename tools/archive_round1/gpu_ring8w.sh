#!/bin/bash
# 8-byte words widened from fp32: the fp64 ring rule on (arm B) vs off
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/ring8w
timeout 1200 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --reps 5 --env TT_KNOB_SD_RING8W=1 > gpurun_out/ring8w/ab.txt 2>&1
