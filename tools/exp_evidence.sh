#!/bin/bash
# round evidence: tests, bench, ncu launch list of the bench command, ncu --set full of the
# C2 Q=4096 s=100% main pass and of the finalize kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out; P=${PFX:-ev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${P}_smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/${P}_pytest.log 2>&1; echo "PYTEST_EXIT $?" >> $O/${P}_pytest.log
timeout 400 python bench.py > $O/${P}_bench_c2.json 2> $O/${P}_bench_c2.err
timeout 400 python bench.py --steps 2 --warmup 3 --no-parity --no-cpu-baseline > $O/${P}_bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|gather|tc_topk|threshold|finalize|f32_to_bf16" -s 200 -c 700 --csv --log-file $O/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-parity --no-cpu-baseline > $O/${P}_ncu_launch.log 2>&1
timeout 120 python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_topk|finalize|threshold" -s 0 -c 4 -o $O/${P}_c2big python tools/run_cell.py --sel 1.0 --q 4096 --reps 1 --graph 0 > $O/${P}_ncu_full.log 2>&1
echo done
for w in c1 c5; do
  timeout 900 python bench.py --workload $w > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err
done
for w in c3 c4; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err
done
echo done2
