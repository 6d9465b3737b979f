#!/bin/bash
# batch B: parity + the C2 cells after the epilogue / finalize rewrite
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-b}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for s in 0.001 0.01 0.1 1.0; do for q in 1 16 256 4096; do timeout 120 python tools/run_cell.py --sel $s --q $q >> $O/${P}_cells.txt 2>&1; done; done
for s in 0.001 0.1 1.0; do timeout 120 python tools/run_cell.py --sel $s --q 1 --path 2 >> $O/${P}_cells.txt 2>&1; done
for s in 0.1 1.0; do timeout 120 python tools/run_cell.py --sel $s --q 4096 --prec 1 >> $O/${P}_cells.txt 2>&1; done
VRS_EPI_SKIP=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 >> $O/${P}_cells.txt 2>&1
VRS_STATS=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_stats.txt 2>&1
VRS_STATS=1 timeout 120 python tools/run_cell.py --sel 0.1 --q 4096 --reps 1 --graph 0 >> $O/${P}_stats.txt 2>&1
timeout 300 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_topk -s 1 -c 1 -o $O/${P}_tc_main python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu.log 2>&1
echo done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:finalize -s 0 -c 1 -o $O/${P}_fin python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_fin.log 2>&1
