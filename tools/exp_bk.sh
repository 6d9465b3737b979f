#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bk}
timeout 1100 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for e in "" "VRS_NO_CPGATHER=1"; do
  for c in "0.001 1" "0.01 16" "0.1 1" "0.1 16"; do set -- $c
    env $e timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
  done
  env $e timeout 300 python tools/run_cell.py --workload c4 --n 6250000 --sel 0.05 --q 1 | sed "s/^/[$e] /" >> $O/${P}_ab.txt 2>&1
done
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
for w in c3 c4; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err; done
echo done
