#!/bin/bash
# probe density for large d (MMA-bound main pass: the epilogue has slack)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ap}
for st in 8 16 32; do
  VRS_PROBE_STEP=$st timeout 300 python tools/run_cell.py --workload c3 --sel 1.0 --q 1024 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
  VRS_PROBE_STEP=$st timeout 300 python tools/run_cell.py --workload c3 --sel 0.1 --q 1024 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
  VRS_PROBE_STEP=$st timeout 600 python tools/run_cell.py --workload c4 --n 6250000 --sel 0.5 --q 8192 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
  VRS_PROBE_STEP=$st timeout 600 python tools/run_cell.py --workload c4 --n 6250000 --sel 0.05 --q 8192 | sed "s/^/[step $st] /" >> $O/${P}_ab.txt 2>&1
done
echo done
