cd "$GRAFT_REPO_ROOT"
ncu --set full --clock-control none --import-source on -k regex:tile -s 2 -c 1 -o gpurun_out/sdsrc python tools/run_case.py "46,46,46,46,46" "3,1,0,4,2" 8 3 > gpurun_out/sdsrc.log 2>&1
ncu -i gpurun_out/sdsrc.ncu-rep --page source --csv --print-source sass > gpurun_out/sdsrc.src.csv 2>/dev/null
ncu -i gpurun_out/sdsrc.ncu-rep --page raw --csv > gpurun_out/sdsrc.raw.csv 2>/dev/null
rm -f gpurun_out/sdsrc.ncu-rep
