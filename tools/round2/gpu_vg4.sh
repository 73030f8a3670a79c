set -x
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vector_gather" 2>&1 | tail -3
timeout 300 python tools/plan_time_probe.py > gpurun_out/plan_time_probe.jsonl 2>&1; head -3 gpurun_out/plan_time_probe.jsonl
timeout 1200 python tools/ab_vg.py --suite s3,set2 --per-cell 1 --variants vg3,vg4,vg3p1 --out gpurun_out/ab_vg4.jsonl 2>&1 | tail -4
O=gpurun_out/vgncu4; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for c in "5,5,5,5,5,5,5,5,5,5,5,5 0,8,4,10,1,3,9,5,7,2,6,11 4" "5,3,2,4,35,33,37,40 7,6,5,4,3,2,1,0 4"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_vg -s 2 -c 1 -o $O/vg python tools/run_case.py $c 3 vector_gather=1 stages=3 > /dev/null 2>&1
  python tools/ncu_summary.py $O/vg.ncu-rep >> $O/summary.txt 2>&1
  ncu -i $O/vg.ncu-rep --page source --csv > $O/vg_source_$(echo $c | cut -c1-5).csv 2>/dev/null; rm -f $O/vg.ncu-rep
done
