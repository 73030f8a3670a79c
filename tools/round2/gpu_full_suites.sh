cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2full; mkdir -p $O
( time timeout 6000 python bench.py --suites full --suites-plan both-all --steps 20 --warmup 5 --no-e2e --suites-out $O/suites_full_cases.jsonl > $O/bench_full.json 2> $O/bench_full.err ) 2> $O/time.txt
tail -c 1500 $O/bench_full.json; tail -3 $O/bench_full.err; cat $O/time.txt
