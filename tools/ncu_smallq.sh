# ncu --set full of the first 30 kernels of a small-batch cell (eager launches: the first search is
# cold, the later ones repeat it), for the HBM-bound cells; then the same cells timed without ncu.
# usage (on the GPU box): bash tools/ncu_smallq.sh
set -x
for cell in "c3 1.0 1" "c4 0.5 1" "c4 0.05 1" "c3 0.1 64"; do
  set -- $cell
  tag=${1}_s${2}_q${3}
  python tools/run_cell.py --workload $1 --sel $2 --q $3 --reps 2 > gpurun_out/s5_cell_$tag.txt 2>&1
  timeout 900 ncu --set full --clock-control none -c 30 \
    -k regex:'select|gather|tc_topk|threshold|finalize|exact' -f -o gpurun_out/s5_ncu_$tag \
    python tools/run_cell.py --workload $1 --sel $2 --q $3 --reps 1 --graph 0 > gpurun_out/s5_ncu_$tag.log 2>&1
done
