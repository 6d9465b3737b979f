#!/bin/bash
# per-CTA timelines of the tensor-core passes (libvrs_exp built with -DVRS_TC_TIMING)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-tl}
for c in "1.0 4096" "0.1 4096" "1.0 256" "0.01 16" "0.001 1"; do set -- $c
  VRS_LIB=exp timeout 120 python tools/tc_timeline.py --sel $1 --q $2 >> $O/${P}_timeline.txt 2>&1
done
echo done
