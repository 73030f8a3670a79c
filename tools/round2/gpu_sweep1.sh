cd "$GRAFT_REPO_ROOT"
timeout 2400 python tools/vg_tile_sweep.py profiles/round2_checkpoint2/suites_cases.jsonl 12 > gpurun_out/vg_tile_sweep.jsonl 2>&1
tail -12 gpurun_out/vg_tile_sweep.jsonl | cut -c1-600
