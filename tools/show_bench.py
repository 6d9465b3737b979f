"""Print a bench JSON line compactly: python tools/show_bench.py file.json"""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "no json:", e)
        continue
    print(f"== {path}: value {d['value']:.4g} {d['unit']} ms/step {d['ms_per_step']:.3f} e2e {d['e2e']['value']:.4g} "
          f"launches {d['gpu_launches']} dtype {d['dtype']}")
    r = d.get("roofline") or {}
    if r:
        print(f"   roofline {r['kernel']}: {r['achieved']:.1f}/{r['peak']:.1f} {r['unit']} frac {r['frac']:.3f}")
    c = d.get("cpu_baseline") or {}
    print(f"   cpu {c.get('value')} cores {c.get('cores')} parity {(d.get('parity') or {}).get('ok')} clocks {d['clocks']}")
    print("   kernels ms/step", {k: round(v, 3) for k, v in d.get("kernels_ms_per_step", {}).items()})
    for c in d.get("cells", []):
        print(f"   s={c['sel']:<8g} q={c['q']:<5d} nsel={c['n_sel']:<9d} {c['ms']:8.3f} ms {c['qps']:12.0f} q/s "
              f"hbm={c['hbm_frac']:.2f} tc={c.get('tensor_frac', c.get('tensor_frac_burst', 0)):.2f}")
