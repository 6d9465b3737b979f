"""Per-CTA timeline of one search's kernels (debug build only).

Build: make -C paper_2403_15807_b200/csrc exp EXP_FLAGS=-DVRS_TC_TIMING, then
  VRS_LIB=exp python tools/tc_timeline.py --sel 1.0 --q 4096
Stamps (globaltimer, ns): 0 entry, 1 after griddepcontrol.wait, 5 CTA end; the
tensor-core passes add 2 first stage landed (MMA warp), 3 first accumulator
ready (epilogue), 4 epilogue done.  First: the whole chain, one line per kernel.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2403_15807_b200 as vrs  # noqa: E402
from paper_2403_15807_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--sel", type=float, default=1.0)
ap.add_argument("--q", type=int, default=4096)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--graph", type=int, default=1, help="time a CUDA-graph replay of the search (as bench.py does)")
a = ap.parse_args()
cfg = datagen.CONFIGS[a.workload]
n = a.n or cfg.n
X, attrs = datagen.corpus(cfg, 0, n, "cuda", n=n)
Q = datagen.queries(cfg, a.q, "cuda")
ix = vrs.Index(X, attrs)
pred = datagen.predicate(cfg, a.sel)
lib = ctypes.CDLL(_lib.LIB_PATH)
fn = lib.vrs_debug_timeline
fn.argtypes = [ctypes.c_int, ctypes.c_void_p]
bufs = [np.zeros((8, 4096, 8), dtype=np.uint64) for _ in range(3)]
out = (torch.empty(a.q, cfg.k, dtype=torch.int64, device="cuda"), torch.empty(a.q, cfg.k, device="cuda"))
run = lambda: ix.search(Q, pred, k=cfg.k, metric=cfg.metric, out=out)  # noqa: E731
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    for _ in range(3):
        run()
torch.cuda.current_stream().wait_stream(st)
torch.cuda.synchronize()
if a.graph:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    run = g.replay
for _ in range(3):
    run()
torch.cuda.synchronize()
for tu in range(3):
    fn(tu, bufs[tu].ctypes.data)
run()
torch.cuda.synchronize()
for tu in range(3):
    assert fn(tu, bufs[tu].ctypes.data) == 0
KNAMES = {(0, 0): "select_count", (0, 1): "select_scatter", (1, 0): "tc main", (1, 1): "tc probe",
          (1, 4): "gather_copy", (1, 5): "f32_to_bf16", (1, 6): "select_finish", (2, 0): "threshold",
          (2, 1): "finalize", (2, 2): "merge"}
rows = []
for (tu, r), name in KNAMES.items():
    b = bufs[tu][r].astype(np.int64)
    b = b[b[:, 0] > 0]
    if len(b):
        rows.append((b[:, 0].min(), name, b))
t0 = min(r[0] for r in rows)
print(f"== chain cell {a.workload} sel={a.sel} q={a.q} {'graph' if a.graph else 'eager'} (us from the first kernel entry; per kernel: CTAs, "
      f"first entry, last past-wait, last end, median in-kernel after the wait)")
for _, name, b in sorted(rows, key=lambda r: r[0]):
    end = b[:, 5]
    print(f"   {name:15s} {len(b):5d} CTAs  entry {(b[:, 0].min() - t0) / 1e3:7.1f}  waited {(b[:, 1].max() - t0) / 1e3:7.1f}"
          f"  end {(end.max() - t0) / 1e3:7.1f}  work {np.median(end - b[:, 1]) / 1e3:6.2f}", end="")
    if name in ("threshold", "finalize") and (b[:, 2] > 0).all():   # inner stamps 2-4 (thread 0)
        inner = [np.median(b[:, i + 1] - b[:, i]) / 1e3 for i in range(1, 5) if (b[:, i + 1] > 0).all()]
        print("  [steps " + " ".join(f"{x:.2f}" for x in inner) + "]", end="")
    print()
buf = bufs[1]
names = {0: "main", 1: "probe"}
t_origin = None
for mode in (1, 0):
    b = buf[mode].astype(np.int64)
    used = b[:, 0] > 0
    if not used.any():
        continue
    b = b[used]
    if t_origin is None:
        t_origin = b[:, 0].min()
    us = lambda x: x / 1000.0  # noqa: E731
    st = b[:, :6] - t_origin
    print(f"== {names[mode]} cell {a.workload} sel={a.sel} q={a.q}: {len(b)} CTAs, tiles/CTA "
          f"{b[:, 7].min()}..{b[:, 7].max()}, span {us(st[:, 5].max() - st[:, 0].min()):.1f} us "
          f"(first entry {us(st[:, 0].min()):.1f}, last end {us(st[:, 5].max()):.1f})")
    d = np.diff(b[:, :6], axis=1)
    labels = ["pdl wait", "first stage", "first acc", "tile loop", "drain"]
    for i, lab in enumerate(labels):
        print(f"   {lab:12s} median {us(np.median(d[:, i])):8.2f}  min {us(d[:, i].min()):8.2f}  max {us(d[:, i].max()):8.2f} us")
    loop = d[:, 3] / np.maximum(b[:, 7], 1)
    print(f"   per tile (loop / tiles) median {us(np.median(loop)):.3f} us, min {us(loop.min()):.3f}, max {us(loop.max()):.3f}")
    # waves: CTAs per SM in start order
    sm = b[:, 6]
    order = np.argsort(st[:, 0])
    waves = {}
    for i in order:
        waves.setdefault(int(sm[i]), []).append(i)
    depth = max(len(v) for v in waves.values())
    print(f"   SMs used {len(waves)}, max CTAs per SM {depth}")
    for w in range(depth):
        idx = [v[w] for v in waves.values() if len(v) > w]
        e = st[idx]
        print(f"   wave {w}: {len(idx)} CTAs, start {us(e[:, 0].min()):.1f}..{us(e[:, 0].max()):.1f}, "
              f"loop start(med) {us(np.median(e[:, 3])):.1f}, end {us(e[:, 5].min()):.1f}..{us(e[:, 5].max()):.1f} us")
