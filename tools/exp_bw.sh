#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bw}
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_range.py tests/test_gpu_parity.py -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
PFX=$P bash tools/exp_bs.sh
