cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_rowtile2; mkdir -p $O
timeout 2400 python tools/ab_opts.py --suite s3,set2 --per-cell 20 --kernel-filter rowcopy --reps 5 kernel=2 > $O/ab_tile.txt 2>&1; tail -6 $O/ab_tile.txt
