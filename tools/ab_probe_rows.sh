# A/B of partial probe tiles (VRS_PROBE_ROWS) on the small-batch cells that fetch rows by cp.async,
# then parity with the switch on (cp.async forced so that small test shapes take the partial tiles).
for cell in c4:0.05:1 c4:0.5:1 c3:0.1:1 c4:0.05:8 c3:0.015625:1; do
  IFS=: read wl sel q <<< "$cell"
  n=""; [ "$wl" = c4 ] && n="--n 6250000"
  for v in - VRS_PROBE_ROWS=128 VRS_PROBE_ROWS=64 VRS_PROBE_ROWS=32; do
    envs=""; [ "$v" != "-" ] && envs="$v"
    echo -n "[$v] "
    env $envs timeout 300 python tools/run_cell.py --workload $wl --sel $sel --q $q $n --reps 2 2>&1 | grep '^cell' | cut -c1-330
  done
done
echo "== parity, VRS_PROBE_ROWS=64 VRS_CPGATHER=1"
VRS_PROBE_ROWS=64 VRS_CPGATHER=1 python -m pytest tests/test_gpu_ar8.py tests/test_gpu_exact.py "tests/test_gpu_fuzz.py::test_fuzz_parity_large_d" -q 2>&1 | tail -3
echo "== parity, VRS_PROBE_ROWS=64, full size"
VRS_PROBE_ROWS=64 python -m pytest tests/test_gpu_fullsize.py -q 2>&1 | tail -3
