#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bg}
for st in 1 2 4 8; do
  VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
  VRS_STATS=1 VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 2>&1 | grep "mode=0" | sort | uniq -c | sed "s/^/[step $st] /" >> $O/${P}_ab.txt
done
VRS_EPI_SKIP=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[skip] /" >> $O/${P}_ab.txt 2>&1
echo done
