#!/bin/bash
# option sweeps and an ncu capture of the worst generic-tile suite cases
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/worst
O=gpurun_out/worst
C1="5,5,5,5,5,5,5,5,5,5,5,5 0,8,4,10,1,3,9,5,7,2,6,11 4"
C2="3,6,6,6,6,6,6,6,6,6,6 0,7,2,3,6,9,10,8,5,1,4 4"
C3="5,3,2,4,35,33,37,40 7,6,5,4,3,2,1,0 4"
timeout 300 python tools/case_sweep.py $C1 "slot_dims=1" "slot_dims=-1" "slots=8" "slots=4" "run_in=32,run_out=128" "run_in=32,run_out=256" "run_in=128,run_out=64" "ctas_per_sm=1" "ctas_per_sm=3" > $O/c1.txt 2>&1
timeout 300 python tools/case_sweep.py $C2 "slot_dims=1" "slots=8" "slots=4" "run_in=32,run_out=128" "run_in=32,run_out=256" "threads=512" "ctas_per_sm=1" "ctas_per_sm=3" > $O/c2.txt 2>&1
timeout 300 python tools/case_sweep.py $C3 "slot_dims=1" "slot_dims=-1" "slots=8" "slots=4" "run_in=32,run_out=32" "ctas_per_sm=1" "ctas_per_sm=3" > $O/c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile -s 2 -c 1 -o $O/c2 python tools/run_case.py "3,6,6,6,6,6,6,6,6,6,6" "0,7,2,3,6,9,10,8,5,1,4" 4 3 > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py $O/c2.ncu-rep > $O/c2_summary.txt 2>&1
ncu -i $O/c2.ncu-rep --page raw --csv > $O/c2_raw.csv 2>/dev/null
ncu -i $O/c2.ncu-rep --page source --csv > $O/c2_source.csv 2>/dev/null
rm -f $O/c2.ncu-rep
