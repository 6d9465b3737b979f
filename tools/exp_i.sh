#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-i}
for st in 16 32 8; do
  for c in "1.0 4096" "0.1 4096" "1.0 256" "1.0 16"; do set -- $c
    VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[step $st] /" >> $O/${P}_cells.txt 2>&1
  done
done
VRS_STATS=1 VRS_PROBE_STEP=32 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_stats.txt 2>&1
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"finalize|threshold" -c 2 -o $O/${P}_fin python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu.log 2>&1
echo done
