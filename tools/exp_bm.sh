#!/bin/bash
# 2 cp.async producer warps (default) vs 1 (libvrs_exp), forced cp.async at every size
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bm}
VRS_CPGATHER=1 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_range.py -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
timeout 900 python -m pytest tests/test_gpu_optin.py -x -q >> $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp default exp; do
  for c in "0.0001 1" "0.015625 1" "0.015625 64" "0.1 1" "0.1 64"; do set -- $c
    VRS_LIB=$lib VRS_CPGATHER=1 timeout 300 python tools/run_cell.py --workload c3 --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  for c in "0.01 16" "0.1 16"; do set -- $c
    VRS_LIB=$lib VRS_CPGATHER=1 timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done
for c in "0.0001 1" "0.015625 1" "0.015625 64" "0.1 1" "0.1 64"; do set -- $c
  VRS_NO_CPGATHER=1 timeout 300 python tools/run_cell.py --workload c3 --sel $1 --q $2 | sed "s/^/[copy] /" >> $O/${P}_ab.txt 2>&1
done
echo done
