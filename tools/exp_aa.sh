#!/bin/bash
# per-lane slow path (default) vs warp-voted group loop (libvrs_exp: -DVRS_SLOW_GROUPS_VOTE)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-aa}
PFX=$P bash tools/exp_m.sh
for s in 0.001 0.01 0.1 1.0; do
  VRS_LIB=exp timeout 120 python tools/run_cell.py --sel $s --q 4096 | sed "s/^/[vote] /" >> $O/${P}_ab.txt 2>&1
  VRS_LIB=exp timeout 120 python tools/run_cell.py --sel $s --q 256 | sed "s/^/[vote] /" >> $O/${P}_ab.txt 2>&1
done
for s in 0.1 0.3; do
  timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 >> $O/${P}_ab.txt 2>&1
  VRS_LIB=exp timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[vote] /" >> $O/${P}_ab.txt 2>&1
done
for s in 0.01 0.1; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$s.csv python tools/run_cell.py --sel $s --q 4096 --reps 1 --graph 0 > /dev/null 2>&1
done
echo done
