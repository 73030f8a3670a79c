cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_rowrule2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 2400 python tools/ab_suite.py build/ab/libtt_rule1.so --suite s2,s3,set2 --per-cell 8 --reps 5 > $O/ab.txt 2>&1; tail -14 $O/ab.txt
