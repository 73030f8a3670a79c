#!/bin/bash
# slot-dim map with a cp.async ring (TT_KNOB_SD_STAGES): parity, then same-box A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/sdasync
O=gpurun_out/sdasync
for S in 3 4; do
  TT_KNOB_SD_STAGES=$S timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x \
    -k "slot_dim or shapes or random_suite_scaled or set2 or ttc_suite or exhaustive_tiny or classification" > $O/parity_$S.txt 2>&1
done
timeout 300 python tools/case_sweep.py "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4 > $O/c1_default.txt 2>&1
TT_KNOB_SD_STAGES=3 timeout 300 python tools/case_sweep.py "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4 "slot_dims=1" "run_in=32,run_out=128" > $O/c1_s3.txt 2>&1
TT_KNOB_SD_STAGES=4 timeout 300 python tools/case_sweep.py "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4 "slot_dims=1" "run_in=32,run_out=128" > $O/c1_s4.txt 2>&1
TT_KNOB_SD_STAGES=3 timeout 300 python tools/case_sweep.py "3,6,6,6,6,6,6,6,6,6,6" "0,7,2,3,6,9,10,8,5,1,4" 4 "slot_dims=1" > $O/c2_s3.txt 2>&1
for S in 3 4; do
  timeout 1200 python tools/ab_opts.py --suite s3,set2 --per-cell 1 --reps 5 --env TT_KNOB_SD_STAGES=$S > $O/ab_$S.txt 2>&1
done
