"""Host-side cost of one search call (no synchronisation inside the loop): the Python
binding vs the bare C call, torch's caching allocator vs libvrs's own pool."""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_2403_15807_b200 as vrs  # noqa: E402
from paper_2403_15807_b200 import _lib  # noqa: E402

cfg = datagen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = min(cfg.n, 2_000_000)
X, attrs = datagen.corpus(cfg, 0, n, "cuda", n=n)
Q = datagen.queries(cfg, 1, "cuda")
pred = datagen.predicate(cfg, cfg.sels[0])
lib = vrs.library()


def per_call(fn, reps=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    return t


for alloc in ("torch", None):
    ix = vrs.Index(X, attrs, allocator=alloc)
    out = (torch.empty(1, cfg.k, dtype=torch.int64, device="cuda"), torch.empty(1, cfg.k, device="cuda"))
    t_py = per_call(lambda: ix.search(Q, pred, k=cfg.k, metric=["l2", "ip", "cos"][cfg.metric], out=out))
    pr, keep = _lib.make_predicate(pred)
    args = (ix._h, ctypes.c_void_p(Q.data_ptr()), 1, cfg.d, ctypes.byref(pr), cfg.k, cfg.metric,
            ctypes.c_void_p(out[0].data_ptr()), ctypes.c_void_p(out[1].data_ptr()), None,
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    t_c = per_call(lambda: lib.vrs_search_ex(*args))
    print(f"{cfg.name} allocator={alloc}: binding {t_py:.1f} us/call, bare C call {t_c:.1f} us/call, "
          f"launches {vrs.last_launches()}")
    del ix
