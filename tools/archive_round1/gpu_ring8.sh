#!/bin/bash
# fp64 rule: slot-dim cp.async ring at one CTA/SM. Arm B = rule off (TT_KNOB_SD_RING8=0):
# ratio > 1 means the rule (arm A, the default) is faster.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/ring8
O=gpurun_out/ring8
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 3 --reps 5 --env TT_KNOB_SD_RING8=0 > $O/ab_off.txt 2>&1
