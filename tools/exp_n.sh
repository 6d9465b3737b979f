#!/bin/bash
# probe on/off for the small batches
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-n}
for v in "" "VRS_NO_PROBE=1"; do
  for s in 0.001 0.01 0.1 1.0; do for q in 1 16 256; do
    env $v timeout 120 python tools/run_cell.py --sel $s --q $q | sed "s/^/[$v] /" >> $O/${P}_cells.txt 2>&1
  done; done
done
VRS_NO_PROBE=1 VRS_STATS=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 16 --reps 1 --graph 0 > $O/${P}_stats.txt 2>&1
echo done
