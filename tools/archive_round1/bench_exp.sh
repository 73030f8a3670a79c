cd "$GRAFT_REPO_ROOT"
for i in 1 2 3; do python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('run', j['value'], j['frac_of_memcpy'], j['memcpy_gbs_per_gpu'], j['roofline']['traffic'])"; done
