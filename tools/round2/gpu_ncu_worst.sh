cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ncu_worst; mkdir -p $O
python tools/first_plan_probe.py > $O/first_plan_lazy.json 2>&1; cat $O/first_plan_lazy.json
CUDA_MODULE_LOADING=EAGER python tools/first_plan_probe.py > $O/first_plan_eager.json 2>&1; cat $O/first_plan_eager.json
C="10,9,23,2,11,9,26,9,2 4,6,0,3,7,2,8,1,5 4"
for v in heur alt; do
  opts=""; [ $v = alt ] && opts="run_in=10 run_out=2860"
  python tools/run_case.py $C 20 $opts > $O/run_$v.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile -s 2 -c 1 -o $O/w_$v python tools/run_case.py $C 3 $opts > $O/ncu_$v.log 2>&1
  python tools/ncu_summary.py $O/w_$v.ncu-rep > $O/w_${v}_summary.txt 2>&1
  ncu -i $O/w_$v.ncu-rep --page raw --csv > $O/w_${v}_raw.csv 2>/dev/null
  rm -f $O/w_$v.ncu-rep
done
