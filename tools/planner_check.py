"""Planner check: the AUTO plan of every bench cell against every forced choice.

For each cell (selectivity, Q) of a workload, times (CUDA-graph replay of one search, median of
`--reps`) the library's own choice and the forced alternatives it chooses between:
  auto        -- the planner (vrs_api.cu row_plan + the tensor-core / scan dispatch)
  masked      -- every row streams, unqualified rows masked (VRS_ROWS_MASKED)
  gather      -- the selection delivered gathered, the library's copy / cp.async rule (VRS_ROWS_GATHER)
  copy        -- gathered through the X_sel copy only (VRS_NO_CPGATHER=1, its own process)
  cpasync     -- gathered by cp.async by id for any size / query-tile count (its own process)
  scan        -- the per-tuple scan path over the 16-bit shadow (VRS_PATH_SCAN)
and reports auto / best (auto: the better of the planner's two runs, first and last process).  One process per environment variant (the switches are read once).

    python tools/planner_check.py --workload c4 > profiles/r02_planner_c4.txt
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# one process per variant: a variant that loads the GPU for long (masked streams every row)
# would otherwise lower the clocks (1 kW power cap) under the next variant's timing
ENV_VARIANTS = {
    "auto": {}, "masked": {}, "gather": {}, "scan": {},
    "copy": {"VRS_NO_CPGATHER": "1"},
    "cpasync": {"VRS_CP_QTILES": "1000000", "VRS_CP_MIN_MB": "0"},
    "auto2": {},   # the planner again, last: process-order effects show as auto != auto2
}


def worker(workload, variant, reps):
    import torch

    import datagen
    import paper_2403_15807_b200 as vrs
    cfg = datagen.CONFIGS[workload]
    r0, r1, _ = datagen.rows_of(cfg, 1, 0)
    X, attrs = datagen.corpus(cfg, r0, r1, "cuda")
    Q = datagen.queries(cfg, max(cfg.qs), "cuda")
    ix = vrs.Index(X, attrs)
    opts = {"auto": [("auto", {})], "auto2": [("auto2", {})], "masked": [("masked", {"rows": vrs.ROWS_MASKED})],
            "gather": [("gather", {"rows": vrs.ROWS_GATHER})], "scan": [("scan", {"path": vrs.PATH_SCAN})],
            "copy": [("copy", {"rows": vrs.ROWS_GATHER})],
            "cpasync": [("cpasync", {"rows": vrs.ROWS_GATHER})]}[variant]
    out = {}
    for s in cfg.sels:
        pred = datagen.predicate(cfg, s)
        for q in cfg.qs:
            graphs = {}
            for name, kw in opts:
                if name == "scan" and q > 64:
                    continue
                res = (torch.empty(q, cfg.k, dtype=torch.int64, device="cuda"), torch.empty(q, cfg.k, device="cuda"))
                try:
                    run = lambda: ix.search(Q[:q], pred, k=cfg.k, metric=cfg.metric, out=res, **kw)  # noqa: E731
                    st = torch.cuda.Stream()
                    st.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(st):
                        run()
                    torch.cuda.current_stream().wait_stream(st)
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        run()
                    g.replay()
                    torch.cuda.synchronize()
                    graphs[name] = (g, res)
                except Exception as e:   # noqa: BLE001
                    out[f"{s}|{q}|{name}"] = None
                    print(f"# {name} s={s} q={q}: {e}", file=sys.stderr)
            ts = {name: [] for name in graphs}
            for name, (g, _r) in graphs.items():
                for i in range(reps + 3):   # (3 warm-up replays)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    g.replay()
                    b.record()
                    torch.cuda.synchronize()
                    if i >= 3:
                        ts[name].append(a.elapsed_time(b))
            for name, v in ts.items():
                v.sort()
                out[f"{s}|{q}|{name}"] = v[len(v) // 2]
            del graphs
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--worker", default=None)
    a = ap.parse_args()
    if a.worker:
        worker(a.workload, a.worker, a.reps)
        return
    res = {}
    for v, env in ENV_VARIANTS.items():
        e = dict(os.environ, **env)
        p = subprocess.run([sys.executable, __file__, "--workload", a.workload, "--reps", str(a.reps), "--worker", v],
                           env=e, capture_output=True, text=True)
        if p.returncode != 0:
            print(f"# worker {v} failed: {p.stderr[-2000:]}")
            continue
        res.update(json.loads(p.stdout.strip().splitlines()[-1]))
    import datagen
    cfg = datagen.CONFIGS[a.workload]
    names = ["auto", "auto2", "masked", "gather", "copy", "cpasync", "scan"]
    print(f"# planner check, workload {a.workload} (one search per cell, CUDA-graph replay, median of {a.reps}, ms)")
    print("| s | Q | " + " | ".join(names) + " | best forced | auto / best |")
    print("|---|---|" + "---|" * (len(names) + 2))
    worst = 0.0
    for s in cfg.sels:
        for q in cfg.qs:
            row = [res.get(f"{s}|{q}|{n}") for n in names]
            forced = [t for n, t in zip(names, row) if n not in ("auto", "auto2") and t is not None]
            best = min(forced) if forced else None
            auto = min(t for t in row[:2] if t is not None) if any(t is not None for t in row[:2]) else None
            ratio = auto / best if auto and best else float("nan")
            worst = max(worst, ratio if ratio == ratio else 0.0)
            cells = " | ".join("-" if t is None else f"{t:.3f}" for t in row)
            print(f"| {s:g} | {q} | {cells} | {best:.3f} | {ratio:.3f} |")
    print(f"\nworst auto / best forced: {worst:.3f}")


if __name__ == "__main__":
    main()
