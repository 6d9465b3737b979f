#!/bin/bash
# full bench on every workload (1 GPU)
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-d}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
for w in c1 c5 c3 c4; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err
done
echo done
