#!/bin/bash
# round 2, late: compute-sanitizer over the code changed late in the round --
# the vector-gather kernels (new item arithmetic, 3-item and 85-register
# instantiations), the 2-D fallback, and the chunked NCCL exchange
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/san3; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="vector_gather or fallback or misaligned or test_shapes"
timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$SEL" > $O/memcheck_vg.txt 2>&1; echo "rc=$?" >> $O/memcheck_vg.txt
timeout 1500 $CS --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "vector_gather" > $O/synccheck_vg.txt 2>&1; echo "rc=$?" >> $O/synccheck_vg.txt
timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$SEL" > $O/initcheck_vg.txt 2>&1; echo "rc=$?" >> $O/initcheck_vg.txt
timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider -k "chunked or redistribution" > $O/memcheck_chunked.txt 2>&1; echo "rc=$?" >> $O/memcheck_chunked.txt
for f in $O/*.txt; do echo "== $f"; tail -3 $f; done
