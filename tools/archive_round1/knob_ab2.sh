#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/pytest_parity_rule.txt 2>&1
run() { env "$@" timeout 900 python bench_suite.py --suite s2,s3,set2 --per-cell 1 --reps 7 --verify none --out gpurun_out/kab_$tag.jsonl > /dev/null 2>&1; }
tag=B1 run TT_KNOB_PREFIX_TARGETS=0
tag=R1 run TT_KNOB_PREFIX_TARGETS=-1
tag=B2 run TT_KNOB_PREFIX_TARGETS=0
tag=R2 run TT_KNOB_PREFIX_TARGETS=-1
