#!/bin/bash
# compute-sanitizer memcheck over a small GPU test subset (one tool per call)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-k}
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -x -q -k "not config_shaped" > $O/${P}_memcheck.log 2>&1
echo "EXIT $?" >> $O/${P}_memcheck.log
