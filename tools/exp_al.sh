#!/bin/bash
# one-wave probe (<= 148 / qtiles splits) vs the main pass's splits
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-al}
PFX=$P bash tools/exp_m.sh
for c in "0.001 4096" "0.01 4096" "0.1 4096" "1.0 4096"; do set -- $c
  VRS_PROBE_FULLP=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[fullp] /" >> $O/${P}_ab.txt 2>&1
done
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_ab.txt 2>&1
  VRS_PROBE_FULLP=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[fullp] /" >> $O/${P}_ab.txt 2>&1
done
for s in 0.1 1.0; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$s.csv python tools/run_cell.py --sel $s --q 4096 --reps 1 --graph 0 > /dev/null 2>&1
done
echo done
