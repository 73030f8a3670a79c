cd "$GRAFT_REPO_ROOT"
bash tools/gpu_sanitize_r2.sh > gpurun_out/san2_run.log 2>&1; tail -20 gpurun_out/san2_run.log
O=gpurun_out/r2check4; mkdir -p $O
( time timeout 2400 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 600 $O/bench.json; tail -3 $O/bench.err; cat $O/bench_time.txt
