#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/fillb
timeout 900 python tools/ab_opts.py --suite s2,s3,set2,s4 --per-cell 3 --reps 7 --env TT_KNOB_T2D_FILLB4=1.0 \
    > gpurun_out/fillb/ab_e4_1.0.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/fillb/parity.txt 2>&1
