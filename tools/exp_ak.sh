#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ak}
for s in 0.01 0.1 1.0; do
  echo "== sel $s" >> $O/${P}_stats.txt
  VRS_STATS=1 timeout 120 python tools/run_cell.py --sel $s --q 4096 --reps 1 --graph 0 2>&1 | sort | uniq -c >> $O/${P}_stats.txt
  VRS_EPI_SKIP=1 timeout 120 python tools/run_cell.py --sel $s --q 4096 | sed "s/^/[episkip] /" >> $O/${P}_stats.txt 2>&1
done
echo done
