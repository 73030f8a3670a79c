cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_rowrule; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 1800 python tools/ab_suite.py build/ab/libtt_prerow.so --suite s2,s3,set2 --per-cell 6 --reps 7 > $O/ab.txt 2>&1; tail -14 $O/ab.txt
