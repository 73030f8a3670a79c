#!/bin/bash
# held-out check of the widened-row rule: arm B = the old 512 B threshold
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/rowmin
timeout 1200 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --reps 5 --env TT_KNOB_ROW_MIN_W=512 \
    > gpurun_out/rowmin/ab_heldout_old.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rowmin/pytest_gpu.txt 2>&1
