#!/bin/bash
# A/B of the default build vs the experiment build (VRS_LIB=exp) on the key C2 cells
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-x}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp; do
  for c in "1.0 4096" "0.1 4096" "0.01 4096" "1.0 256" "1.0 16" "0.1 16" "1.0 1" "0.01 1"; do
    set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_cells.txt 2>&1
  done
done
VRS_STATS=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_stats.txt 2>&1
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_topk -s 1 -c 1 -o $O/${P}_tc_main python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu.log 2>&1
VRS_LIB=exp timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_topk -s 1 -c 1 -o $O/${P}_tc_main_exp python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_exp.log 2>&1
echo done
