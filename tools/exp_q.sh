#!/bin/bash
# gathered-row norms A/B follow-up: C2 grid + C5 mid cells
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-q}
PFX=$P bash tools/exp_m.sh
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_cells.txt 2>&1
done
echo done
