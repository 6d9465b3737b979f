#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bl}
timeout 1100 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for e in "" "VRS_NO_CPGATHER=1"; do
  for c in "0.0001 1" "0.015625 1" "0.015625 64" "0.1 1" "0.1 64"; do set -- $c
    env $e timeout 300 python tools/run_cell.py --workload c3 --sel $1 --q $2 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
  done
  for s in 0.001 0.05; do env $e timeout 300 python tools/run_cell.py --workload c4 --n 6250000 --sel $s --q 1 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1; done
done
for w in c2 c3 c4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err; done
echo done
