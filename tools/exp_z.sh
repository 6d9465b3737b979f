#!/bin/bash
# masked vs gathered rows at high selectivity: epilogue stats
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-z2}
for c in "0.9 4096" "0.5 4096" "1.0 4096"; do set -- $c
  for r in 1 2; do
    echo "== sel $1 q $2 rows $r" >> $O/${P}_stats.txt
    VRS_STATS=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 --rows $r --reps 1 --graph 0 2>&1 | sort | uniq -c >> $O/${P}_stats.txt
  done
done
echo done
