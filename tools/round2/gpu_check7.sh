cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "measured" > $O/pytest_measured.txt 2>&1; tail -2 $O/pytest_measured.txt
( time timeout 3000 python bench.py --suites-plan both-all --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 300 $O/bench.json; tail -3 $O/bench.err; cat $O/bench_time.txt
