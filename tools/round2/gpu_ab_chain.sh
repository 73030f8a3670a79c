cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_chain; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 1500 python tools/ab_suite.py build/ab/libtt_base.so --suite s2,s3,set2 --per-cell 1 --reps 7 > $O/ab.txt 2>&1; tail -20 $O/ab.txt
