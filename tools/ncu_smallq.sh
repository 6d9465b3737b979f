# ncu --set full of the first 30 kernels of a small-batch cell (eager launches: the first search is
# cold, the later ones repeat it), for the HBM-bound cells; then the same cells timed without ncu.
# usage (on the GPU box): bash tools/ncu_smallq.sh
set -x
for cell in "c3 1.0 1" "c4 0.5 1" "c4 0.05 1" "c3 0.1 64"; do
  set -- $cell
  tag=${1}_s${2}_q${3}
  n=""; [ "$1" = c4 ] && n="--n 6250000"
  python tools/run_cell.py --workload $1 --sel $2 --q $3 --reps 2 $n > gpurun_out/s5_cell_$tag.txt 2>&1
  timeout 900 ncu --set full --clock-control none -c 16 \
    -k regex:'select|gather|tc_topk|threshold|finalize|exact' -f -o gpurun_out/s5_ncu_$tag \
    python tools/run_cell.py --workload $1 --sel $2 --q $3 --reps 1 --graph 0 $n > gpurun_out/s5_ncu_$tag.log 2>&1
  # (the reports are 60+ MB each: summarise on the box, bring back the markdown only)
  python tools/ncu_summary.py gpurun_out/s5_ncu_$tag.ncu-rep "$1 s=$2 Q=$3, first 16 kernels of the process (two searches, eager)" > gpurun_out/s5_ncu_$tag.md 2>> gpurun_out/s5_ncu_$tag.log
  rm -f gpurun_out/s5_ncu_$tag.ncu-rep
done
