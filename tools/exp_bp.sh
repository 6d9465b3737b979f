#!/bin/bash
# slow-path appends from registers (default) vs staged + serial loop (libvrs_exp: -DVRS_STAGED_APPEND)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bp}
timeout 1100 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp default exp; do
  for c in "0.01 4096" "0.1 4096" "1.0 4096" "1.0 256"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
done
for lib in default exp; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
echo done
