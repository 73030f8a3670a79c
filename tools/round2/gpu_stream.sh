cd "$GRAFT_REPO_ROOT"
timeout 900 python tools/ab_streaming.py gpurun_out/ab_streaming.jsonl 2>&1 | tail -25
