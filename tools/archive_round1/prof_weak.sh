#!/bin/bash
# ncu --set full on the weakest single-GPU classes (one launch each)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/weak
run() {  # name dims perm esize
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:'tile|tiled2d|rowcopy' -s 2 -c 1 \
     -o gpurun_out/weak/$1 python tools/run_case.py "$2" "$3" $4 3 > gpurun_out/weak/$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/weak/$1.ncu-rep > gpurun_out/weak/$1.txt 2>&1
  ncu -i gpurun_out/weak/$1.ncu-rep --page source --csv > gpurun_out/weak/$1.src.csv 2>/dev/null
  rm -f gpurun_out/weak/$1.ncu-rep
}
run s2r3_585 "585,585,585" "1,0,2" 8
run s2r4_119 "119,119,119,119" "3,2,1,0" 8
run set2r8 "5,3,2,4,35,33,37,40" "7,6,5,4,3,2,1,0" 4
run s3r12 "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4
run s2r6_46 "36,77,15,5,51,19" "4,3,2,5,0,1" 8
