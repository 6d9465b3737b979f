#!/bin/bash
# scan path (per-tuple FFMA over the compacted selection) vs tensor-core path on small batches
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ac}
for s in 0.001 0.01 0.1 1.0; do for q in 1 16 64 256; do
  timeout 120 python tools/run_cell.py --sel $s --q $q --path 1 | sed "s/^/[scan] /" >> $O/${P}_cells.txt 2>&1
done; done
for c in "0.001 1" "0.01 16" "1.0 16"; do set -- $c
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$1_$2.csv python tools/run_cell.py --sel $1 --q $2 --path 1 --reps 1 --graph 0 > /dev/null 2>&1
done
echo done
