#!/bin/bash
# mid-size gathered cell (C2 s=0.1 q=4096): epilogue stats, launch list, ncu full of probe/main
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-r}
for s in 0.1 1.0; do
VRS_STATS=1 timeout 120 python tools/run_cell.py --sel $s --q 4096 --reps 1 --graph 0 >> $O/${P}_stats.txt 2>&1
done
timeout 120 python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_topk" -s 0 -c 4 -o $O/${P}_mid python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_full.log 2>&1
echo done
