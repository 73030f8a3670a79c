cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_unroll; mkdir -p $O
python tools/first_plan_probe.py > $O/first_plan.json 2>&1; cat $O/first_plan.json
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 1500 python tools/ab_suite.py build/ab/libtt_unrolled.so --suite s2,s3,set2 --per-cell 2 --reps 7 > $O/ab.txt 2>&1; tail -14 $O/ab.txt
