#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/sdasync2
O=gpurun_out/sdasync2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "slot_dim or measured" > $O/parity.txt 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "slot_dim_async" > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "slot_dim_async" > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 1500 python bench_suite.py --suite s3,set2 --per-cell 1 --plan both --verify sampled --out $O/suites_both.jsonl > /dev/null 2> $O/suites.err
