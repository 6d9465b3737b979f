#!/bin/bash
# small-cell chain anatomy: default / no probe+threshold / no PDL
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ar}
for c in "0.001 1" "0.01 16" "0.001 256"; do set -- $c
  timeout 120 python tools/run_cell.py --sel $1 --q $2 >> $O/${P}_ab.txt 2>&1
  VRS_NO_PROBE=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[noprobe] /" >> $O/${P}_ab.txt 2>&1
  VRS_NO_PDL=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[nopdl] /" >> $O/${P}_ab.txt 2>&1
done
echo done
