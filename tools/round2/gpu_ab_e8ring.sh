cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_e8ring; mkdir -p $O
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 2 --kernel-filter tile --esize 8 slot_dims=1 stages=4 > $O/ab_sd4.txt 2>&1; tail -6 $O/ab_sd4.txt
timeout 1500 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 2 --kernel-filter tile --esize 8 vector_gather=1 stages=3 > $O/ab_vg3.txt 2>&1; tail -6 $O/ab_vg3.txt
timeout 1500 python tools/ab_opts.py --suite s3,set2 --per-cell 2 --kernel-filter tile --esize 4 slot_dims=1 stages=4 > $O/ab_e4_sd4.txt 2>&1; tail -6 $O/ab_e4_sd4.txt
timeout 1500 python tools/ab_opts.py --suite s3,set2 --per-cell 2 --kernel-filter tile --esize 4 slot_dims=1 stages=3 > $O/ab_e4_sd3.txt 2>&1; tail -6 $O/ab_e4_sd3.txt
