#!/bin/bash
# experiment batch A: C2 Q=4096 s=100% cell variants + TF32 peak + ncu full of the main tensor-core pass
cd $GRAFT_REPO_ROOT
O=gpurun_out
python tools/measure_tf32.py > $O/a_tf32.json 2>&1
for v in "" "VRS_EPI_SKIP=1" "VRS_NO_PROBE=1" "VRS_NO_SAMPLE=1 VRS_NO_PROBE=1" "VRS_PAIR=1" "VRS_TWO_PART=1"; do
  echo "== $v" >> $O/a_cells.txt
  env $v timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 >> $O/a_cells.txt 2>&1
done
for s in 0.001 0.01 0.1; do timeout 120 python tools/run_cell.py --sel $s --q 4096 >> $O/a_cells.txt 2>&1; done
for q in 1 16 256; do timeout 120 python tools/run_cell.py --sel 1.0 --q $q >> $O/a_cells.txt 2>&1; done
VRS_STATS=1 timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/a_stats.txt 2>&1
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/a_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_topk -s 2 -c 1 -o $O/a_tc_main python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/a_ncu.log 2>&1
echo done
