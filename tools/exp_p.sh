#!/bin/bash
# minimum tiles per split A/B on mid-size cells
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-p}
for ms in 4 16 32; do
  for c in "0.01 4096" "0.1 4096" "1.0 4096" "0.1 256" "1.0 256"; do set -- $c
    VRS_MIN_SPAN=$ms timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[span $ms] /" >> $O/${P}_cells.txt 2>&1
  done
  for s in 0.1 0.3; do
    VRS_MIN_SPAN=$ms timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[span $ms] /" >> $O/${P}_cells.txt 2>&1
  done
done
echo done
