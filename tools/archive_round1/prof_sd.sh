cd "$GRAFT_REPO_ROOT"
# slot-dim vs classic generic tile on a case where the slot-dim map lost
for v in 0 -1; do
  ncu --set full --clock-control none -k regex:tile -s 2 -c 1 -o gpurun_out/sd_$v python tools/run_case.py "46,46,46,46,46" "3,1,0,4,2" 8 3 slot_dims=$v > gpurun_out/sd_$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/sd_$v.ncu-rep > gpurun_out/sd_$v.txt 2>&1
  rm -f gpurun_out/sd_$v.ncu-rep
done
for v in 0 -1; do
  ncu --set full --clock-control none -k regex:tile -s 2 -c 1 -o gpurun_out/sdw_$v python tools/run_case.py "7,4,11,14,12,3,12,5,5,3" "0,6,8,1,3,5,4,9,2,7" 4 3 slot_dims=$v > gpurun_out/sdw_$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/sdw_$v.ncu-rep > gpurun_out/sdw_$v.txt 2>&1
  rm -f gpurun_out/sdw_$v.ncu-rep
done
