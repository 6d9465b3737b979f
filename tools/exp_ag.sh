#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ag}
for b in 296 592 1184; do
for c in "0.001 1" "0.01 16" "0.1 256" "0.1 4096"; do set -- $c
  VRS_FINISH_BLOCKS=$b timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[fin $b] /" >> $O/${P}_ab.txt 2>&1
done
VRS_FINISH_BLOCKS=$b timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[fin $b] /" >> $O/${P}_ab.txt 2>&1
done
for c in "0.001 1" "0.01 16" "0.1 256" "0.1 4096"; do set -- $c
  VRS_SELECT_SCATTER=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[scatter] /" >> $O/${P}_ab.txt 2>&1
done
VRS_SELECT_SCATTER=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[scatter] /" >> $O/${P}_ab.txt 2>&1
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
timeout 400 python bench.py --workload c1 --steps 5 --warmup 3 > $O/${P}_bench_c1.json 2> $O/${P}_bench_c1.err
echo done
