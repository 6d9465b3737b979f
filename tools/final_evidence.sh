# Round-end evidence: bench lines for every workload, the reference arm, smoke and the C4
# launch list (ncu, cold-cache serialised launches: compare shares), into gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1
for w in c4 c1 c2 c3 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/fin_bench_$w.json 2> gpurun_out/fin_bench_$w.err
done
timeout 900 python bench.py --impl reference > gpurun_out/fin_bench_c4_reference.json 2> gpurun_out/fin_bench_c4_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/fin_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-parity --no-cpu-baseline --no-cells > gpurun_out/fin_ncu_bench.log 2>&1
