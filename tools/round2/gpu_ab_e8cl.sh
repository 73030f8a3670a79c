# slot-dim and vector-gather load phases vs the heuristic's classic tile on fp64 perm[0] != 0 cases
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/abe8; mkdir -p $O
timeout 1800 python tools/ab_vg.py --suite s3,set2,s2 --per-cell 3 --perm0 nonzero --esize 8 --kind classic --variants sd,sd3,vg3,vg4 --out $O/ab_e8cl.jsonl > $O/e8cl.log 2>&1
tail -5 $O/e8cl.log
