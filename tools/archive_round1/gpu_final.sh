#!/bin/bash
# round checkpoint: smoke, all GPU tests, headline bench (+ reference arm),
# fused-P2P bench config on one GPU, ncu launch list + full capture of S1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config s5p2p --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_s5p2p.json 2> $O/bench_s5p2p.err
timeout 600 python bench.py --config s5redist --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_s5local1.json 2> $O/bench_s5local1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_s1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled2d -s 3 -c 1 -o $O/prof_s1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/prof_s1.ncu-rep > $O/prof_s1.txt 2>&1
ncu -i $O/prof_s1.ncu-rep --page raw --csv > $O/prof_s1_raw.csv 2>/dev/null
rm -f $O/prof_s1.ncu-rep
