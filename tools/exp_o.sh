#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-o}
for s in 0.001 1.0; do for q in 1 16 256 4096; do
  timeout 120 python tools/run_cell.py --sel $s --q $q >> $O/${P}_cells.txt 2>&1
done; done
echo done
