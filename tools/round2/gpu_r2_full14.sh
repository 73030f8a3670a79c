cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2full14; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
( time timeout 6000 python bench.py --suites full --suites-plan both-all --steps 20 --warmup 5 --no-e2e --no-order-check --suites-out $O/suites_full_cases.jsonl > $O/bench_full.json 2> $O/bench_full.err ) 2> $O/full_time.txt
tail -c 600 $O/bench_full.json; cat $O/full_time.txt
