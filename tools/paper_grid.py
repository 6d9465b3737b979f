"""The paper's own filtered-scan grid (Sec. 5, Figs. 7-8) on this library, for context:
1M tuples, vectors and one relational column uniformly random, D in {64, 1024},
query batch in {1, 10000}, selectivity 1 / 10 / 50 / 100 %, "cosine similarity > 0.9"
(vrs_range_search) and top-64 (vrs_search, k = 64 as in the paper's index runs, L350).
The paper's CPU times (2x Xeon Gold 5118, 48 threads) are printed beside.
    python tools/paper_grid.py > profiles/rNN_paper_grid.txt"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_15807_b200 as vrs  # noqa: E402

# PAPER.md L1059-L1364 (Figs. 7-8): best of Scan / Tensor, ms per batch
PAPER = {(64, 1): {0.01: 0.677, 0.10: 2.04, 0.50: 5.02, 1.0: 7.41},
         (1024, 1): {0.01: 1.25, 0.10: 8.81, 0.50: 37.4, 1.0: 67.9},
         (64, 10000): {0.01: 31.7, 0.10: 303.5, 0.50: 1513.3, 1.0: 2855.7},
         (1024, 10000): {0.01: 398.9, 0.10: 3767.3, 0.50: 11195.3, 1.0: 23289.0}}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


def main():
    n = 1_000_000
    g = torch.Generator(device="cuda")
    g.manual_seed(2403)
    print("D  batch  sel   | range cos>0.9: ms  results/q | top-64: ms | paper best (CPU, 48 thr) ms | speed-up (top-64)")
    for d in (64, 1024):
        X = torch.rand(n, d, device="cuda", generator=g) * 2 - 1
        attr = torch.randint(0, 100, (n,), device="cuda", dtype=torch.int32, generator=g)
        ix = vrs.Index(X, [attr])
        for b in (1, 10000):
            Q = torch.rand(b, d, device="cuda", generator=g) * 2 - 1
            for s in (0.01, 0.10, 0.50, 1.0):
                pred = [(0, 0, int(round(s * 100)) - 1)]
                tr, (off, ids, _) = timed(lambda: ix.range_search(Q, pred, tau=0.9, metric="cos"))
                tk, _ = timed(lambda: ix.search(Q, pred, k=64, metric="cos"))
                p = PAPER[(d, b)][s]
                print(f"{d:<4} {b:<6} {s:<5} | {tr:10.3f} {ids.numel() / b:10.2f} | {tk:9.3f} | {p:12.2f} | "
                      f"{p / tk:9.1f}x", flush=True)
        del ix, X


if __name__ == "__main__":
    main()
