#!/bin/bash
# per-CTA timelines of one search's kernels (libvrs_exp built with -DVRS_TC_TIMING);
# CELLS="sel,q sel,q ..." (default: five C2 cells); TL_ARGS: extra tc_timeline.py flags
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-tl}
for c in ${CELLS:-1.0,4096 0.1,4096 1.0,256 0.01,16 0.001,1}; do
  IFS=, read sel q <<< "$c"
  VRS_LIB=exp timeout 120 python tools/tc_timeline.py --sel $sel --q $q $TL_ARGS >> $O/${P}_timeline.txt 2>&1
done
echo done
