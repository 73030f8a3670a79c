cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_l2pf; mkdir -p $O
for pf in 128B 256B; do
  timeout 1500 python tools/ab_suite.py build/ab/libtt_sd_$pf.so --suite s3,set2 --per-cell 2 --reps 7 > $O/ab_$pf.txt 2>&1; tail -12 $O/ab_$pf.txt
done
