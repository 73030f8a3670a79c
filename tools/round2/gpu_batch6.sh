cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2check5; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
timeout 1200 python tools/ab_tma.py $O/ab_tma.jsonl > /dev/null 2>&1; tail -4 $O/ab_tma.jsonl
( time timeout 3000 python bench.py --suites-out $O/suites_cases.jsonl > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
tail -c 400 $O/bench.json; tail -3 $O/bench.err; cat $O/bench_time.txt
cuobjdump -sass paper_1705_01598_b200/libtt.so | grep -oE "UTMALDG|UTMASTG|UBLKCP|LDGSTS|UTC[A-Z]*MMA" | sort | uniq -c > $O/sass_counts.txt; cat $O/sass_counts.txt
