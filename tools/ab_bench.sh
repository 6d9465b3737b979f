# A/B of environment switches on whole bench steps (no parity / CPU baseline).
# usage: bash tools/ab_bench.sh <workload> "<variants: NAME=V,NAME2=V2 | - ...>" [steps]
wl=$1; steps=${3:-10}
for v in $2; do
  envs=""; [ "$v" != "-" ] && envs=$(echo "$v" | tr ',' ' ')
  env $envs python bench.py --workload $wl --steps $steps --warmup 3 --no-cpu-baseline --no-parity > /tmp/ab_bench.json 2> /tmp/ab_bench.err || tail -5 /tmp/ab_bench.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("/tmp/ab_bench.json").read().strip().splitlines()[-1])
k = {n: round(x, 3) for n, x in d.get("kernels_ms_per_step", {}).items()}
print(f"[{sys.argv[1]}] {d['value']:.0f} {d['unit']}  {d['ms_per_step']:.3f} ms/step  clocks {d['clocks'].get('sm_mhz')}  cert {d.get('certificate')}  {k}")
PY
done
