#!/bin/bash
# ASan + UBSan over the host code (planner and oracle); logs in profiles/sanitizer/
set -e
cd "$(dirname "$0")"
OUT=../../profiles/sanitizer
mkdir -p $OUT /tmp/tt_san
g++ -std=c++17 -g -O1 -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -I/usr/local/cuda/include planner_fuzz.cpp ../../paper_1705_01598_b200/csrc/planner.cpp -o /tmp/tt_san/planner_fuzz
gcc -std=c99 -g -O1 -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -ffp-contract=off oracle_fuzz.c ../../oracle/tt_oracle.c -o /tmp/tt_san/oracle_fuzz
( /tmp/tt_san/planner_fuzz; echo "exit $?" ) > $OUT/asan_ubsan_planner.txt 2>&1
( /tmp/tt_san/oracle_fuzz; echo "exit $?" ) > $OUT/asan_ubsan_oracle.txt 2>&1
cat $OUT/asan_ubsan_planner.txt $OUT/asan_ubsan_oracle.txt
