#!/bin/bash
# round checkpoint: smoke, GPU tests, headline bench, suites (verified), one
# ncu capture of the slot-dim tile kernel on a SET2 case
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke3.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu3.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 1200 python bench_suite.py --suite s2,s3,set2,s4 --per-cell 1 --out gpurun_out/suite21.jsonl > /dev/null 2> gpurun_out/suite21.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_sd -s 2 -c 1 -o gpurun_out/sd_set2 python tools/run_case.py "5,3,2,4,35,33,37,40" "7,6,5,4,3,2,1,0" 4 3 > gpurun_out/sd_set2.log 2>&1
python tools/ncu_summary.py gpurun_out/sd_set2.ncu-rep > gpurun_out/sd_set2.txt 2>&1
rm -f gpurun_out/sd_set2.ncu-rep
