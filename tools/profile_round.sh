#!/bin/bash
# ncu evidence for the round (run under gpurun; single GPU, never multi-rank).
#   launch list of bench.py (cold-cache, serialised: compare shares, not absolutes)
#   --set full capture of the dominant kernel of each bench config
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_s1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/launches_s1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiled2d -s 3 -c 1 \
    -o gpurun_out/full_s1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full_s1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 3 -c 1 \
    -o gpurun_out/full_s2 python bench.py --config s2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full_s2.log 2>&1
python tools/ncu_summary.py gpurun_out/full_s1.ncu-rep > gpurun_out/full_s1.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_s2.ncu-rep > gpurun_out/full_s2.txt 2>&1
