#!/bin/bash
# main-pass split count for Q = 4096 (qtiles 32): P 18 (default: 576 CTAs, 3.9 waves) vs 23 (736, 4.97) vs 37 (1184, 8.0)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-pq}
for rep in 1 2; do for pp in 18 23 37; do
  for c in "1.0 4096" "0.1 4096" "0.01 4096"; do set -- $c
    VRS_P=$pp timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[P$pp] /" >> $O/${P}_ab.txt 2>&1
  done
done; done
echo done
