#!/bin/bash
# same-box A/B of the prefix run targets (timing only, verification in tests)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
run() { env "$@" timeout 900 python bench_suite.py --suite s2,s3,set2 --per-cell 1 --reps 7 --verify none --out gpurun_out/kab_$tag.jsonl > /dev/null 2>&1; }
tag=B1 run TT_KNOB_PREFIX_TARGETS=0
tag=A1 run TT_KNOB_PREFIX_TARGETS=1
tag=B2 run TT_KNOB_PREFIX_TARGETS=0
tag=A2 run TT_KNOB_PREFIX_TARGETS=1
