cd "$GRAFT_REPO_ROOT"
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/h_r12 python tools/run_case.py "5,5,5,5,5,5,5,5,5,5,5,5" "0,8,4,10,1,3,9,5,7,2,6,11" 4 3 > gpurun_out/h_r12.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/h_set2 python tools/run_case.py "5,3,2,4,35,33,37,40" "7,6,5,4,3,2,1,0" 4 3 > gpurun_out/h_set2.log 2>&1
for f in h_r12 h_set2; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/$f.src.csv 2>/dev/null; done
rm -f gpurun_out/h_r12.ncu-rep gpurun_out/h_set2.ncu-rep
