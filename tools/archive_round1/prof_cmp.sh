cd "$GRAFT_REPO_ROOT"
# fp64 11584^2: 2-D vector kernel vs generic tile, same problem
ncu --set full --clock-control none --import-source on -k regex:tiled2d -s 2 -c 1 -o gpurun_out/c_t2d python tools/run_case.py "11584,11584" "1,0" 8 3 > gpurun_out/c_t2d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/c_gen python tools/run_case.py "11584,11584" "1,0" 8 3 kernel=2 run_in=32 run_out=32 > gpurun_out/c_gen.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 -o gpurun_out/c_gen2 python tools/run_case.py "11584,11584" "1,0" 8 3 kernel=2 run_in=64 run_out=64 threads=512 > gpurun_out/c_gen2.log 2>&1
for f in c_t2d c_gen c_gen2; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; done
