#!/bin/bash
# re-entry checkpoint: smoke, GPU tests (incl. strided plans), headline bench, suites
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke4.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu4.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench4_ref.json 2> gpurun_out/bench4_ref.err
timeout 1200 python bench_suite.py --suite s2,s3,set2,s4 --per-cell 1 --out gpurun_out/suite4.jsonl > /dev/null 2> gpurun_out/suite4.err
