cd "$GRAFT_REPO_ROOT"
timeout 900 python tools/measure_probe.py 2,3,4,3,2,2,3,2,20,18,22,24 7,0,2,8,10,5,9,4,6,11,1,3 4 > gpurun_out/measure_probe.jsonl 2>&1
sort -t: -k2 -n -r gpurun_out/measure_probe.jsonl | head -12; tail -1 gpurun_out/measure_probe.jsonl
