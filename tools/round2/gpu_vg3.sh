set -x
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/vgpol; mkdir -p $O
C1="5,5,5,5,5,5,5,5,5,5,5,5 0,8,4,10,1,3,9,5,7,2,6,11 4"
C3="5,3,2,4,35,33,37,40 7,6,5,4,3,2,1,0 4"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for c in 1 3; do
  eval C=\$C$c
  timeout 300 ncu --metrics $M --clock-control none -k regex:tile -s 2 -c 1 --csv python tools/run_case.py $C 3 > $O/c${c}_heur.csv 2>&1
  for pol in 0 1 2 3; do
    timeout 300 ncu --metrics $M --clock-control none -k regex:tile -s 2 -c 1 --csv python tools/run_case.py $C 3 vector_gather=1 stages=4 vg_policy=$pol > $O/c${c}_vg_p$pol.csv 2>&1
  done
done
timeout 1200 python tools/ab_vg.py --suite s3,set2 --per-cell 1 --variants vg3,vg4,vg3p1,vg4p1,vg3p2,vg4p2,vg4p3 --out gpurun_out/ab_vg3.jsonl 2>&1 | tail -8
