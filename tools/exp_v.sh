#!/bin/bash
# launch lists of small cells (serialised kernel durations) + bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-v2}
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
for c in "0.001 1" "0.01 16" "0.1 256" "1.0 16" "0.01 4096"; do set -- $c
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$1_$2.csv python tools/run_cell.py --sel $1 --q $2 --reps 1 --graph 0 > /dev/null 2>&1
done
VRS_EPI_SKIP=1 timeout 120 python tools/run_cell.py --sel 0.1 --q 4096 > $O/${P}_episkip.txt 2>&1
echo done
