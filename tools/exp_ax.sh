#!/bin/bash
# big cell anatomy: full / read-out only / no epilogue
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ax}
for m in 0 2 1; do
  if [ $m = 0 ]; then E=""; else E="VRS_EPI_SKIP=$m"; fi
  env $E timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[epi $m] /" >> $O/${P}_ab.txt 2>&1
  env $E timeout 120 python tools/run_cell.py --sel 0.1 --q 4096 | sed "s/^/[epi $m] /" >> $O/${P}_ab.txt 2>&1
done
echo done
