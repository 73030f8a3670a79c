#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu5.txt 2>&1
timeout 900 python bench_suite.py --suite s2,s4 --per-cell 1 --out gpurun_out/suite5.jsonl > /dev/null 2> gpurun_out/suite5.err
