#!/bin/bash
# device-side probe density + finalize ncu (C2 s=0.1 q=4096)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-t2}
PFX=$P bash tools/exp_m.sh
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_cells.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"finalize" -s 0 -c 1 -o $O/${P}_fin python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_full.log 2>&1
echo done
