#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-f3}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for c in "1.0 4096" "0.1 4096" "0.01 4096"; do set -- $c
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_l_$1_$2.csv python tools/run_cell.py --sel $1 --q $2 --reps 1 --graph 0 > /dev/null 2>&1
done
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
echo done
