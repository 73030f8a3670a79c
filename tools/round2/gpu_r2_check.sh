# round-2 checkpoint: GPU tests, smoke, default bench (with suites), launch list
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check; mkdir -p $O
nproc > $O/nproc.txt
( time timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1 ) 2> $O/pytest_time.txt
tail -3 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
( time timeout 2400 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 3000 $O/bench.json; tail -5 $O/bench.err
