#!/bin/bash
# finalize_warp_kernel<256,64> register limit: default (8 CTAs/SM) vs libvrs_m6 / libvrs_m4
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-fm}
for rep in 1 2; do for lib in "" m6 m4; do
  for c in "0.01 4096" "0.1 4096" "1.0 4096"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done; done
for lib in "" m6 m4; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
echo done
