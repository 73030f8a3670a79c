#!/bin/bash
# heuristic-plan suites (every case verified against the oracle on sampled positions)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/suites
timeout 2400 python bench_suite.py --suite s2,s3,set2,s4 --per-cell 1 --plan heuristic --out gpurun_out/suites/heuristic.jsonl > /dev/null 2> gpurun_out/suites/heuristic.err
