cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_2dtile; mkdir -p $O
timeout 2400 python tools/ab_opts.py --suite s2,s3,set2,s4 --per-cell 8 --kernel-filter tiled2d --reps 5 kernel=2 > $O/ab_2d_to_tile.txt 2>&1; tail -8 $O/ab_2d_to_tile.txt
timeout 2400 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 8 --kernel-filter tile --reps 5 kernel=4 > $O/ab_tile_to_2d.txt 2>&1; tail -8 $O/ab_tile_to_2d.txt
