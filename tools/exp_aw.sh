#!/bin/bash
# 16 epilogue warps / 4 lists per split (libvrs_exp: -DVRS_LPS=4) vs 8 / 2
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-aw}
VRS_LIB=exp timeout 1100 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_optin.py::test_slow_path_vote_variant > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp; do
  for c in "0.001 4096" "0.01 4096" "0.1 4096" "1.0 4096" "1.0 256" "0.1 256" "1.0 16" "0.01 1"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  for s in 0.1 0.3; do
    VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel $s --q 2048 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c3 --sel 1.0 --q 1024 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
done
VRS_LIB=exp timeout 400 python bench.py > $O/${P}_bench_c2_exp.json 2> $O/${P}_bench_c2_exp.err
echo done
