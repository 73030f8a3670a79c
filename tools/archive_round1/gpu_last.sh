#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/last
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/last/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/last/smoke.txt
timeout 2400 python bench_suite.py --suite s2,s3,set2,s4 --per-cell 1 --plan heuristic --out gpurun_out/last/heuristic.jsonl > /dev/null 2> gpurun_out/last/heuristic.err
