#!/bin/bash
# default bench, libvrs_old vs libvrs_new alternating (same box)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ab2}
for rep in 1 2; do for lib in old new; do
  VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_${lib}_$rep.json 2>&1
done; done
echo done
