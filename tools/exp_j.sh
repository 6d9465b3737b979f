#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-j}
for s in 0.001 0.01 0.1 0.3; do timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_cells.txt 2>&1; done
VRS_EPI_SKIP=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 >> $O/${P}_cells.txt 2>&1
VRS_STATS=1 timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 --reps 1 --graph 0 > $O/${P}_stats.txt 2>&1
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_topk -s 2 -c 1 -o $O/${P}_c5_main python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 --reps 1 --graph 0 > $O/${P}_ncu.log 2>&1
echo done
