#!/bin/bash
# CTA finalize with 16 warps (default) vs 8 (libvrs_exp), alternating
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-bo}
timeout 1100 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
for lib in default exp default exp; do
  for c in "0.001 1" "0.01 16" "0.1 16" "0.1 256" "1.0 1" "1.0 16" "1.0 256"; do set -- $c
    VRS_LIB=$lib timeout 120 python tools/run_cell.py --sel $1 --q $2 | sed "s/^/[$lib] /" >> $O/${P}_ab.txt 2>&1
  done
done
for lib in default exp; do VRS_LIB=$lib timeout 400 python bench.py --no-parity --no-cpu-baseline > $O/${P}_bench_$lib.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:finalize --csv --log-file $O/${P}_l_def.csv python tools/run_cell.py --sel 1.0 --q 16 --reps 1 --graph 0 > /dev/null 2>&1
VRS_LIB=exp timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:finalize --csv --log-file $O/${P}_l_exp.csv python tools/run_cell.py --sel 1.0 --q 16 --reps 1 --graph 0 > /dev/null 2>&1
echo done
