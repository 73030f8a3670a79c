cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check2; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1 ) 2> $O/pytest_time.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python tools/plan_time_probe.py > $O/plan_time_probe.jsonl 2>&1
( time timeout 2400 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 1500 $O/bench.json; tail -5 $O/bench.err
