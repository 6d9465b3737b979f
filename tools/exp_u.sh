#!/bin/bash
# min_p splits + transposed rescore reduction: C2 grid, A/B of min_p on small row spaces
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-u2}
PFX=$P bash tools/exp_m.sh
for c in "0.001 4096" "0.01 4096" "0.001 256" "0.01 256" "0.1 1" "0.01 16"; do set -- $c
  VRS_NO_MIN_P=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[no_min_p] /" >> $O/${P}_ab.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_l.log 2>&1
echo done
