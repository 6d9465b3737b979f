#!/bin/bash
# chunk-level early-out bound (default) vs per-group only (libvrs_exp: -DVRS_NO_CHUNK_BOUND), alternating
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bc}
VRS_LIB=default timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_range.py -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp default exp; do
  for c in "0.1 4096" "1.0 4096" "1.0 256" "1.0 16"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done
for lib in default exp; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
echo done
