cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_2dopts; mkdir -p $O
for o in "stages=-1" "stages=4" "t2d_vec2=1" "t2d_vec2=-1" "ctas_per_sm=3"; do
  f=$(echo $o | tr '=' '_')
  timeout 1200 python tools/ab_opts.py --suite s2,s3,set2,s4 --per-cell 4 --kernel-filter tiled2d --reps 5 $o > $O/ab_$f.txt 2>&1; echo "== $o"; tail -6 $O/ab_$f.txt
done
