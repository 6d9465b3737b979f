#!/bin/bash
# GPU tests + default bench at the working tree
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ck}
timeout 1200 python -m pytest tests -m gpu -q -x > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for i in 1 2; do timeout 400 python bench.py --no-cpu-baseline > $O/${P}_bench_$i.json 2> $O/${P}_bench_$i.err; done
echo done
