#!/bin/bash
# C3 (10M x 768, L2, k=100) big cell: cells + ncu of the main pass
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ao}
for c in "1.0 1024" "0.1 1024" "0.1 1" "0.01 1024"; do set -- $c
  timeout 300 python tools/run_cell.py --workload c3 --sel $1 --q $2 >> $O/${P}_cells.txt 2>&1
done
VRS_STATS=1 timeout 300 python tools/run_cell.py --workload c3 --sel 1.0 --q 1024 --reps 1 --graph 0 2>&1 | sort | uniq -c >> $O/${P}_cells.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_topk" -s 1 -c 1 -o $O/${P}_c3main python tools/run_cell.py --workload c3 --sel 1.0 --q 1024 --reps 1 --graph 0 > $O/${P}_ncu.log 2>&1
echo done
