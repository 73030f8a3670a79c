cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_rowvg; mkdir -p $O
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --kernel-filter rowcopy kernel=2 vector_gather=1 stages=4 > $O/ab_vg4.txt 2>&1; tail -6 $O/ab_vg4.txt
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --kernel-filter rowcopy kernel=2 > $O/ab_tile.txt 2>&1; tail -6 $O/ab_tile.txt
