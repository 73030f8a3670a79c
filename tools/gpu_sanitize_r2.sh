#!/bin/bash
# round 2: compute-sanitizer over the vector-gather kernel (memcheck,
# racecheck, synccheck, initcheck) and initcheck over the small-shape parity
# tests of every kernel family
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/san2; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
VG="vector_gather"
timeout 1200 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$VG" > $O/memcheck_vg.txt 2>&1; echo "rc=$?" >> $O/memcheck_vg.txt
timeout 1200 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$VG" > $O/racecheck_vg.txt 2>&1; echo "rc=$?" >> $O/racecheck_vg.txt
timeout 1200 $CS --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$VG" > $O/synccheck_vg.txt 2>&1; echo "rc=$?" >> $O/synccheck_vg.txt
SEL="s0 or exhaustive_tiny or test_shapes or forced or two_element or async or rowcopy or slot_dim or alignment or misaligned or strided or vector_gather"
timeout 1800 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$SEL" > $O/initcheck.txt 2>&1; echo "rc=$?" >> $O/initcheck.txt
timeout 1200 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "rowcopy or classification" > $O/memcheck_rowcopy.txt 2>&1; echo "rc=$?" >> $O/memcheck_rowcopy.txt
for f in $O/*.txt; do echo "== $f"; tail -3 $f; done
