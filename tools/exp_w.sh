#!/bin/bash
# union-of-top-2 threshold for small batches; finalize_cta ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-w2}
PFX=$P bash tools/exp_m.sh
for c in "0.001 1" "0.1 256" "1.0 16"; do set -- $c
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$1_$2.csv python tools/run_cell.py --sel $1 --q $2 --reps 1 --graph 0 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"finalize" -s 0 -c 1 -o $O/${P}_fincta python tools/run_cell.py --sel 1.0 --q 16 --reps 1 --graph 0 > $O/${P}_ncu_full.log 2>&1
echo done
