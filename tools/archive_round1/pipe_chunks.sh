#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for c in 8 4 16 32 8; do
  TT_KNOB_PIPE_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pipe_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pipe_$c.json')); print($c, d['e2e'])" >> gpurun_out/pipe_chunks.txt
done
