#!/bin/bash
# final check at HEAD: GPU tests, smoke, default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-fin}
timeout 1200 python -m pytest tests -m gpu -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/${P}_smoke.txt 2>&1
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
echo done
