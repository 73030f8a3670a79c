cd "$GRAFT_REPO_ROOT"
# planner knob variants on the same box, suites s2,s3,set2 (no verification: timing only)
run() { env "$@" python bench_suite.py --suite s2,s3,set2 --per-cell 1 --reps 7 --verify none --out gpurun_out/knob_$tag.jsonl > /dev/null 2>&1; }
tag=A run TT_KNOB_PREFIX_TARGETS=1
tag=D run TT_KNOB_PREFIX_TARGETS=0 TT_KNOB_SD_VMAX=4096
tag=B run TT_KNOB_PREFIX_TARGETS=0
tag=C run TT_KNOB_PREFIX_TARGETS=1 TT_KNOB_SD_VMAX=4096
tag=E run TT_KNOB_TILE_LAT=0.75
tag=F run TT_KNOB_TILE_LAT=3.0
tag=A2 run TT_KNOB_PREFIX_TARGETS=1
