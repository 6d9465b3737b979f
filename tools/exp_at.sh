#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-at}
for st in 8 12 16; do for s in 0.01 0.1 0.3; do
  VRS_PROBE_STEP=$st timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
done; done
echo done
