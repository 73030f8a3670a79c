#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu3.txt 2>&1
timeout 2400 python bench_suite.py --suite s2,s3,set2,s4 --per-cell 1 --out $O/suites3.jsonl > /dev/null 2> $O/suites3.err
