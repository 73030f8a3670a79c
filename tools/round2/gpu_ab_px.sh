# vector-gather load phase vs the heuristic plan on perm[0] != 0 tile cases
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/abpx; mkdir -p $O
timeout 1500 python tools/ab_vg.py --suite s3,set2,s2 --per-cell 2 --perm0 nonzero --esize 4 --variants vg3,vg4 --out $O/ab_px_e4.jsonl > $O/e4.log 2>&1
timeout 1200 python tools/ab_vg.py --suite s3,set2,s2 --per-cell 2 --perm0 nonzero --esize 8 --variants vg3,vg4 --out $O/ab_px_e8.jsonl > $O/e8.log 2>&1
tail -3 $O/e4.log $O/e8.log
