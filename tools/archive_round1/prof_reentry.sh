#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
run() {  # name regex dims perm esize
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 2 -c 1 \
     -o $O/$1 python tools/run_case.py "$3" "$4" $5 3 > $O/$1.log 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/$1.txt 2>&1
  rm -f $O/$1.ncu-rep
}
run ring_fp64 tiled2d_sa "31623,6325" "1,0" 8
run scalar_fp32 tiled2d_s "13954,13954" "1,0" 4
run set2_sd tile_sd "5,3,2,4,35,33,37,40" "7,6,5,4,3,2,1,0" 4
run s3r10_prefix "tile" "7,7,7,7,7,7,7,7,7,7" "0,2,1,3,5,4,8,7,9,6" 4
