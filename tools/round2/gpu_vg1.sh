set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vector_gather" 2>&1 | tail -5
timeout 900 python tools/ab_vg.py --suite s3,set2 --per-cell 1 --out gpurun_out/ab_vg1.jsonl 2>&1 | tail -80
