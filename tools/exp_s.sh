#!/bin/bash
# register-only threshold + one-wave finalize; probe step sweep on mid cells
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-s2}
PFX=$P bash tools/exp_m.sh
for st in 2 4 8; do for s in 0.01 0.1 1.0; do
  VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel $s --q 4096 | sed "s/^/[step $st] /" >> $O/${P}_sweep.txt 2>&1
done; done
for st in 4 8 16; do for s in 0.01 0.1 1.0; do
  VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel $s --q 256 | sed "s/^/[step $st] /" >> $O/${P}_sweep.txt 2>&1
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_l.log 2>&1
echo done
