#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "p2p or rowcopy or emulated or nccl" > gpurun_out/pytest_p2p.txt 2>&1
timeout 600 python tools/p2p_emulate.py > gpurun_out/p2p_emulate.jsonl 2> gpurun_out/p2p_emulate.err
