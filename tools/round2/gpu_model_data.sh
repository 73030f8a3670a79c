cd "$GRAFT_REPO_ROOT"
O=gpurun_out/model_data; mkdir -p $O
timeout 2400 python tools/model_data.py --suite s2,s3,set2 --per-cell 2 --out $O/data_train.jsonl > $O/train.log 2>&1; tail -3 $O/train.log
timeout 2400 python tools/model_data.py --suite s3 --per-cell 5 --out $O/data_s3x5.jsonl > $O/s3x5.log 2>&1; tail -3 $O/s3x5.log
