#!/bin/bash
# default vs libvrs_exp (variant named in the call), alternating
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bs}
for lib in default exp default exp; do
  for c in "0.01 4096" "0.1 4096" "1.0 4096" "1.0 256"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
done
for lib in default exp; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
echo done
