#!/bin/bash
# big-cell splits (wave quantisation) and probe density sweep with the per-lane slow path
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ad}
for pp in 18 37 74; do
  VRS_P=$pp timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[P $pp] /" >> $O/${P}_cells.txt 2>&1
done
for st in 6 8 12 16; do
  VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[step $st] /" >> $O/${P}_cells.txt 2>&1
  VRS_P=37 VRS_PROBE_STEP=$st timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 | sed "s/^/[P37 step $st] /" >> $O/${P}_cells.txt 2>&1
done
for dv in 0 4 8 16; do for s in 0.01 0.1; do
  VRS_PROBE_DIV=$dv timeout 120 python tools/run_cell.py --sel $s --q 4096 | sed "s/^/[div $dv] /" >> $O/${P}_cells.txt 2>&1
done; done
for dv in 0 8; do
  VRS_PROBE_DIV=$dv timeout 120 python tools/run_cell.py --sel 1.0 --q 256 | sed "s/^/[div $dv] /" >> $O/${P}_cells.txt 2>&1
done
echo done
