#!/bin/bash
# double-buffered epilogue TMEM loads (libvrs_exp: -DVRS_EPI_DB) vs single
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-au}
for lib in default exp; do
  for c in "0.01 4096" "0.1 4096" "1.0 4096" "1.0 256" "1.0 16"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  for s in 0.1 0.3; do
    VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done
echo done
