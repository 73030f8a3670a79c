#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_contract.py -q -p no:cacheprovider > gpurun_out/pytest_contract.txt 2>&1
timeout 900 python tools/ttgt_bench.py 24 8 > gpurun_out/ttgt_f64.jsonl 2> gpurun_out/ttgt_f64.err
timeout 600 python tools/ttgt_bench.py 12 4 > gpurun_out/ttgt_f32.jsonl 2> gpurun_out/ttgt_f32.err
