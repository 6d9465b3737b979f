#!/bin/bash
# one-kernel selection + select_finish (dense ids / count / gathered rows) vs select_count + select_scatter + gather_copy
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-af}
PFX=$P bash tools/exp_m.sh
for c in "0.001 1" "0.01 16" "0.1 256" "0.1 4096" "1.0 16"; do set -- $c
  VRS_SELECT_SCATTER=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[scatter] /" >> $O/${P}_ab.txt 2>&1
done
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_ab.txt 2>&1
  VRS_SELECT_SCATTER=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[scatter] /" >> $O/${P}_ab.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l.csv python tools/run_cell.py --sel 0.001 --q 1 --reps 1 --graph 0 > /dev/null 2>&1
timeout 900 python bench.py --workload c1 --steps 5 --warmup 3 > $O/${P}_bench_c1.json 2> $O/${P}_bench_c1.err
echo done
