cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_rowcps; mkdir -p $O
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --kernel-filter rowcopy ctas_per_sm=8 > $O/ab_cps8.txt 2>&1; tail -6 $O/ab_cps8.txt
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 6 --kernel-filter rowcopy ctas_per_sm=6 > $O/ab_cps6.txt 2>&1; tail -6 $O/ab_cps6.txt
