#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small-shape GPU parity tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/san
O=gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="s0 or exhaustive_tiny or test_shapes or forced or two_element or async or rowcopy or slot_dim or alignment or misaligned or strided or stream_and_errors"
timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$SEL" > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 1200 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "forced_tiles or forced_tiled2d or slot_dim or async or two_element or s0" > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
timeout 900 $CS --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "forced_tiles or slot_dim or async" > $O/synccheck.txt 2>&1; echo "rc=$?" >> $O/synccheck.txt
timeout 900 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_accumulate.py tests/test_contract.py -m gpu -q -p no:cacheprovider -k "not large" > $O/memcheck_acc_contract.txt 2>&1; echo "rc=$?" >> $O/memcheck_acc_contract.txt
