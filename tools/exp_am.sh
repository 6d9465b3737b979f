#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-am}
for pp in 4 9 18 37; do for s in 0.01 0.1 1.0; do
  VRS_P=$pp timeout 120 python tools/run_cell.py --sel $s --q 4096 | sed "s/^/[P $pp] /" >> $O/${P}_ab.txt 2>&1
done; done
for pp in 37 74 148; do for s in 0.1 1.0; do
  VRS_P=$pp timeout 120 python tools/run_cell.py --sel $s --q 256 | sed "s/^/[P $pp] /" >> $O/${P}_ab.txt 2>&1
done; done
for pp in 9 18 36; do
  VRS_P=$pp timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[P $pp] /" >> $O/${P}_ab.txt 2>&1
done
echo done
