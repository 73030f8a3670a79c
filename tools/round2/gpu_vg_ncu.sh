#!/bin/bash
# ncu --set full of the worst generic-tile case (5^12 fp32) and the Set-2
# rank-8 reversal: heuristic plan vs the vector-gather load phase
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/vgncu
mkdir -p $O
C1="5,5,5,5,5,5,5,5,5,5,5,5 0,8,4,10,1,3,9,5,7,2,6,11 4"
C3="5,3,2,4,35,33,37,40 7,6,5,4,3,2,1,0 4"
for c in 1 3; do
  eval C=\$C$c
  for v in heur vg; do
    opts=""; [ $v = vg ] && opts="vector_gather=1 stages=4"
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile -s 2 -c 1 -o $O/c${c}_$v python tools/run_case.py $C 3 $opts > $O/ncu_c${c}_$v.log 2>&1
    python tools/ncu_summary.py $O/c${c}_$v.ncu-rep > $O/c${c}_${v}_summary.txt 2>&1
    ncu -i $O/c${c}_$v.ncu-rep --page source --csv > $O/c${c}_${v}_source.csv 2>/dev/null
    rm -f $O/c${c}_$v.ncu-rep
  done
done
