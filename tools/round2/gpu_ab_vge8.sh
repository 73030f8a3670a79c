cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_vge8; mkdir -p $O
timeout 2000 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 8 --esize 8 --kernel-filter tile --reps 5 vector_gather=1 stages=4 > $O/ab.txt 2>&1; tail -6 $O/ab.txt
