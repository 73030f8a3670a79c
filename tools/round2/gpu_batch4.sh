cd "$GRAFT_REPO_ROOT"
timeout 1800 python tools/vg_rule_sweep.py 60 gpurun_out/vg_rule_sweep.jsonl > /dev/null 2>&1; tail -8 gpurun_out/vg_rule_sweep.jsonl
bash tools/gpu_ncu_classes.sh > gpurun_out/ncu_classes_run.log 2>&1; tail -40 gpurun_out/ncu_classes_run.log
