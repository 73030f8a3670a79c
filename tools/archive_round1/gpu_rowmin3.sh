#!/bin/bash
# un-widened rows 512 B - 4 KB: row copy (A) vs generic tile incl. the fp64 ring (B)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/rowmin3
timeout 1200 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 3 --reps 5 --env TT_KNOB_ROW_MIN=4096 > gpurun_out/rowmin3/ab.txt 2>&1
