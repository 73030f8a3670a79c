#!/bin/bash
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 600 python bench.py --config s2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench2_s2.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled2d -s 3 -c 1 -o gpurun_out/prof_s1_t2d python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
