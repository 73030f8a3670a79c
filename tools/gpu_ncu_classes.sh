#!/bin/bash
# round 2: ncu --set full of one suite case per kernel class as the planner
# now chooses it; summaries + DRAM traffic per launch
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ncu_classes; mkdir -p $O
timeout 600 python tools/ncu_classes.py > $O/classes.txt 2>&1
cat $O/classes.txt
while read k dims perm e name; do
  [ -z "$name" ] && continue
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile|tiled2d|rowcopy|copy" -s 2 -c 1 -o $O/$k python tools/run_case.py $dims $perm $e 3 > $O/$k.log 2>&1
  echo "case $name dims $dims perm $perm" > $O/${k}_summary.txt
  python tools/ncu_summary.py $O/$k.ncu-rep >> $O/${k}_summary.txt 2>&1
  rm -f $O/$k.ncu-rep
done < $O/classes.txt
for f in $O/*_summary.txt; do echo "== $f"; head -8 $f; done
