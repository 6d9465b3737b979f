#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-h}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for q in 1 64 1024; do timeout 300 python tools/run_cell.py --workload c3 --sel 1.0 --q $q >> $O/${P}_cells.txt 2>&1; done
for q in 1 256; do timeout 300 python tools/run_cell.py --workload c4 --n 6250000 --sel 0.5 --q $q >> $O/${P}_cells.txt 2>&1; done
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
echo done
