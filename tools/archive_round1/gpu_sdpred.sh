#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/pytest_sdpred.txt 2>&1
timeout 1500 python bench_suite.py --suite s3,set2 --per-cell 1 --reps 7 --verify none --out gpurun_out/sdpred.jsonl > /dev/null 2>&1
