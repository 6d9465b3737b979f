#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-m}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for s in 0.001 0.01 0.1 1.0; do for q in 1 16 256 4096; do
  timeout 120 python tools/run_cell.py --sel $s --q $q >> $O/${P}_cells.txt 2>&1
done; done
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
echo done
