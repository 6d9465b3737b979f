"""Run one bench cell a few times (for ncu captures): python tools/run_cell.py --workload c2 --sel 1.0 --q 4096 --reps 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2403_15807_b200 as vrs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--sel", type=float, default=1.0)
ap.add_argument("--q", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--prec", type=int, default=0, help="0 default (the index shadow), 1 tf32, 2 bf16, 3 fp16")
a = ap.parse_args()
cfg = datagen.CONFIGS[a.workload]
n = a.n or cfg.n
X, attrs = datagen.corpus(cfg, 0, n, "cuda", n=n)
Q = datagen.queries(cfg, a.q, "cuda")
ix = vrs.Index(X, attrs)
pred = datagen.predicate(cfg, a.sel)
for _ in range(a.reps):
    ids, d = ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None)
e.record()
torch.cuda.synchronize()
gms = float("nan")
if a.graph:
    out = (torch.empty(a.q, cfg.k, dtype=torch.int64, device="cuda"), torch.empty(a.q, cfg.k, device="cuda"))
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None, out=out)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None, out=out)
    g.replay()
    torch.cuda.synchronize()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    for _ in range(10):
        g.replay()
    e2.record()
    torch.cuda.synchronize()
    gms = s2.elapsed_time(e2) / 10
# host-side cost of one search call (no sync: 40 calls stay within the launch queue)
torch.cuda.synchronize()
import time as _time
t0 = _time.perf_counter()
for _ in range(40):
    ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None)
host_us = (_time.perf_counter() - t0) / 40 * 1e6
torch.cuda.synchronize()
# e2e on host buffers (public call, host_async, pinned): per-call device time incl. H2D / D2H
Qh = Q.cpu().pin_memory()
hid = torch.empty(a.q, cfg.k, dtype=torch.int64, pin_memory=True)
hdi = torch.empty(a.q, cfg.k, dtype=torch.float32, pin_memory=True)
ix.search_host(Qh, pred, k=cfg.k, metric=cfg.metric, out=(hid, hdi), host_async=True)
torch.cuda.synchronize()
s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s3.record()
for _ in range(10):
    ix.search_host(Qh, pred, k=cfg.k, metric=cfg.metric, out=(hid, hdi), host_async=True)
e3.record()
torch.cuda.synchronize()
e2e_ms = s3.elapsed_time(e3) / 10
vrs.profile(True)
vrs.profile_reset()
for _ in range(3):
    ix.search(Q, pred, k=cfg.k, metric=cfg.metric, path=a.path or None, rows=a.rows or None, precision=a.prec or None)
torch.cuda.synchronize()
prof = vrs.profile_read()
vrs.profile(False)
ks = " ".join(f"{k}={v[0]/v[1]*1e3:.0f}us" for k, v in prof.items())
print(f"cell {a.workload} sel={a.sel} q={a.q} prec={vrs.last_precision()}: {s.elapsed_time(e)/3:.3f} ms/search, graph {gms:.3f} ms, host {host_us:.1f} us/call, e2e {e2e_ms:.3f} ms, path={vrs.last_path()} | {ks}")
