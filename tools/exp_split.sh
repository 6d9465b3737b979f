#!/bin/bash
# accumulator released per part (libvrs_split: -DVRS_SPLIT_ACC=1) vs libvrs (per-part barriers,
# whole-tile MMA order) vs libvrs_old (previous HEAD); parity of split and default
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-sp}
VRS_LIB=split timeout 60 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_first.txt 2>&1; echo "FIRST_EXIT $?" >> $O/${P}_first.txt
grep -q "FIRST_EXIT 0" $O/${P}_first.txt || exit 3
for rep in 1 2; do for lib in old "" split; do
  for c in "1.0 4096" "0.1 4096" "1.0 256"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
  VRS_LIB=$lib timeout 300 python tools/run_cell.py --workload c5 --n 2500000 --sel 0.3 --q 2048 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
done; done
for lib in old "" split; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_x$lib.json 2>&1; done
VRS_LIB=split timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py tests/test_gpu_fuzz.py tests/test_gpu_range.py -q -x > $O/${P}_pytest_split.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest_split.log
timeout 1200 python -m pytest tests -m gpu -q -x > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
echo done
