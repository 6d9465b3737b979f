#!/bin/bash
# cp.async gather producer (VRS_CPGATHER) vs the X_sel copy
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bj}
timeout 900 python -m pytest tests/test_gpu_optin.py -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for e in "" "VRS_CPGATHER=1" "" "VRS_CPGATHER=1"; do
  for c in "0.001 1" "0.01 16" "0.1 16" "0.1 256" "0.01 4096" "0.1 4096"; do set -- $c
    env $e timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
  done
  env $e timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
  env $e timeout 300 python tools/run_cell.py --workload c3 --sel 0.1 --q 1 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
  env $e timeout 300 python tools/run_cell.py --workload c3 --sel 0.1 --q 64 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
done
echo done
