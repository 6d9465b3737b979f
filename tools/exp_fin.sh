#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-f2}
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"finalize" -s 0 -c 1 -o $O/${P}_finbig python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_full.log 2>&1
echo done
