cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_sddual; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
timeout 1500 python tools/ab_suite.py build/ab/libtt_vgdual.so --suite s2,s3,set2 --per-cell 4 --reps 7 > $O/ab.txt 2>&1; tail -14 $O/ab.txt
