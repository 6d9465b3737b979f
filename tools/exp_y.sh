#!/bin/bash
# TMA gather4 late materialisation vs the X_sel copy; forced gather vs masked
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-y2}
PFX=$P bash tools/exp_m.sh
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_cells.txt 2>&1
  VRS_GATHER_COPY=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[copy] /" >> $O/${P}_ab.txt 2>&1
done
for c in "0.1 4096" "0.1 16" "0.01 256"; do set -- $c
  VRS_GATHER_COPY=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[copy] /" >> $O/${P}_ab.txt 2>&1
done
for c in "0.3 16" "0.5 16" "0.3 256" "0.5 256" "0.9 4096" "0.5 4096"; do set -- $c
  for r in 1 2; do
    timeout 120 python tools/run_cell.py --sel $1 --q $2 --rows $r | sed "s/^/[rows $r] /" >> $O/${P}_ab.txt 2>&1
  done
done
echo done
