cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_vgs6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vector_gather or shapes or scaled" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 1500 python tools/ab_suite.py build/ab/libtt_s4.so --suite s3,set2 --per-cell 4 --reps 7 > $O/ab.txt 2>&1; tail -12 $O/ab.txt
