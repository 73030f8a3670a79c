cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_vg5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vector_gather or shapes or scaled or full_size" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 1500 python tools/ab_suite.py build/ab/libtt_prevg.so --suite s3,set2 --per-cell 2 --reps 7 > $O/ab.txt 2>&1; tail -12 $O/ab.txt
timeout 600 python tools/ab_opts.py --suite s3,set2 --per-cell 2 --esize 4 --kernel-filter tile vector_gather=1 stages=4 > $O/ab_vg_forced_e4.txt 2>&1; tail -5 $O/ab_vg_forced_e4.txt
