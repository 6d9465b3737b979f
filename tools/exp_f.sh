#!/bin/bash
# PDL A/B on the 16 C2 cells + bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-f}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for v in "" "VRS_NO_PDL=1"; do
  for s in 0.001 0.01 0.1 1.0; do for q in 1 16 256 4096; do
    env $v timeout 120 python tools/run_cell.py --sel $s --q $q | sed "s/^/[$v] /" >> $O/${P}_cells.txt 2>&1
  done; done
done
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
echo done
