cd "$GRAFT_REPO_ROOT"
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/g_r12 python tools/run_case.py "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4 3 > gpurun_out/g_r12.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/g_585 python tools/run_case.py "585,585,585" "2,0,1" 8 3 > gpurun_out/g_585.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/g_set2 python tools/run_case.py "5,3,2,4,35,33,37,40" "7,6,5,4,3,2,1,0" 4 3 > gpurun_out/g_set2.log 2>&1
for f in g_r12 g_585 g_set2; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; done
