#!/bin/bash
# finalize CTA warps (16 below 148 queries): libvrs_old (HEAD~) vs libvrs_new, alternating; then the GPU tests on the new default
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-fw}
for rep in 1 2; do for lib in old new; do
  for c in "0.001 1" "0.01 16" "1.0 16" "0.1 256" "1.0 256" "0.1 4096"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done; done
for lib in old new; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q -x > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
echo done
