cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check18; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
( time timeout 3000 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 400 $O/bench.json; tail -3 $O/bench.err; cat $O/bench_time.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2>&1; tail -c 300 $O/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_s1.csv python bench.py --steps 5 --warmup 3 --suites none --no-cpu-baseline --no-e2e --verify none --no-order-check > $O/ncu_bench.log 2>&1; tail -2 $O/ncu_bench.log
( time timeout 6000 python bench.py --suites full --suites-plan both-all --steps 20 --warmup 5 --no-e2e --no-order-check --suites-out $O/suites_full_cases.jsonl > $O/bench_full.json 2> $O/bench_full.err ) 2> $O/full_time.txt
tail -c 600 $O/bench_full.json; cat $O/full_time.txt
