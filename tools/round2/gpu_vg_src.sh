cd "$GRAFT_REPO_ROOT"
O=gpurun_out/vg_src; mkdir -p $O
C="5,5,5,5,5,5,5,5,5,5,5,5 0,8,4,10,1,3,9,5,7,2,6,11 4"
python tools/run_case.py $C 20 > $O/run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_vg -s 2 -c 1 -o $O/vg python tools/run_case.py $C 3 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/vg.ncu-rep > $O/vg_summary.txt 2>&1
ncu -i $O/vg.ncu-rep --page source --csv --print-source sass > $O/vg_sass.csv 2>/dev/null
ncu -i $O/vg.ncu-rep --page source --csv > $O/vg_src.csv 2>/dev/null
ncu -i $O/vg.ncu-rep --page raw --csv > $O/vg_raw.csv 2>/dev/null
rm -f $O/vg.ncu-rep
ls -la $O
