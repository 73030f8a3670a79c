cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check8; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
( time timeout 3000 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 300 $O/bench.json; tail -3 $O/bench.err; cat $O/bench_time.txt
