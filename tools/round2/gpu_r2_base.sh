set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name())"
( time python bench_suite.py --suite s3,set2 --per-cell 1 --verify full --out gpurun_out/r2_base_s3set2_full.jsonl > gpurun_out/r2_base_s3set2.log 2>&1 ) 2> gpurun_out/r2_base_time.txt
tail -2 gpurun_out/r2_base_s3set2.log
