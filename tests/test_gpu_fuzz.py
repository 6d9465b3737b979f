"""Seeded random shapes against the oracle: n, d, q, k, metric, predicate (0-2
clauses over int32 / uint8 columns, including empty and all-rows), path (auto /
tensor-core / scan), row delivery and selection precision -- the combinations the
hand-written cases do not enumerate.  Same acceptance rule as every parity test."""
import os

import numpy as np
import pytest
import torch

import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu
METRICS = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}
# VRS_FUZZ_BASE shifts every seed (a soak run over fresh cases: VRS_FUZZ_BASE=100000 pytest ...)
SEED_BASE = int(os.environ.get("VRS_FUZZ_BASE", "0"))
N_CASES = 150


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _case(seed):
    rng = np.random.default_rng(SEED_BASE + 1000 + seed)
    n = int(rng.integers(1, 20000))
    d = int(rng.choice([4, 8, 16, 32, 64, 96, 128, 136, 256]))
    q = int(rng.choice([1, 2, 7, 16, 64, 129, 300]))
    k = int(rng.choice([1, 5, 10, 32, 50, 100]))
    metric = int(rng.choice([oracle.L2, oracle.IP, oracle.COS]))
    n_cl = int(rng.integers(0, 3))
    pred = []
    for _ in range(n_cl):
        col = int(rng.integers(0, 2))
        hi_max = 999 if col == 0 else 255
        lo = int(rng.integers(0, hi_max + 1))
        hi = int(rng.integers(lo - 5, hi_max + 1))   # lo > hi sometimes: an empty clause
        pred.append((col, lo, hi))
    path = [None, 2, 1][int(rng.integers(0, 3))]
    rows = [None, 1, 2][int(rng.integers(0, 3))]
    prec = [None, 1, 2, 3][int(rng.integers(0, 4))]
    off = int(rng.integers(0, 1 << 20))
    return rng, n, d, q, k, metric, pred, path, rows, prec, off


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_parity(vrs, seed):
    rng, n, d, q, k, metric, pred, path, rows, prec, off = _case(seed)
    if prec in (2, 3) and d % 8:
        prec = None
    X = rng.standard_normal((n, d)).astype(np.float32)
    if metric == oracle.COS:
        X[np.linalg.norm(X, axis=1) == 0] += 1.0
    attrs = [rng.integers(0, 1000, n).astype(np.int32), rng.integers(0, 256, n).astype(np.uint8)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off,
                   precision=prec)
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=METRICS[metric], path=path, rows=rows)
    torch.cuda.synchronize()
    check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric, row_offset=off)


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_range(vrs, seed):
    """Threshold mode on random shapes: tau between two scores of the first query
    (so result counts vary), ids and offsets exact, dists to fp32 rounding."""
    rng, n, d, q, _, metric, pred, _, rows, prec, off = _case(10_000 + seed)
    if prec in (2, 3) and d % 8:
        prec = None
    q = min(q, 64)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32), rng.integers(0, 256, n).astype(np.uint8)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    _, _, _, sc = oracle.range_search(X, attrs, pred, Q[:1], -np.inf if metric != oracle.L2 else np.inf, metric)
    if len(sc) >= 2:
        s = np.sort(sc)[::-1] if metric != oracle.L2 else np.sort(sc)
        r = int(rng.integers(0, min(len(s) - 1, 200)))
        tau = float((s[r] + s[r + 1]) / 2)
    else:
        tau = 0.0
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off,
                   precision=prec)
    o, ids, dists = ix.range_search(torch.from_numpy(Q).cuda(), pred, tau=tau, metric=METRICS[metric], rows=rows)
    torch.cuda.synchronize()
    ro, rids, rd, _ = oracle.range_search(X, attrs, pred, Q, tau, metric, row_offset=off)
    assert o.cpu().numpy().tolist() == ro.tolist()
    assert ids.cpu().numpy().tolist() == rids.tolist()
    assert np.allclose(dists.cpu().numpy(), rd, rtol=1e-6, atol=1e-7)


N_CASES_LARGE_D = 80


def _case_large_d(seed):
    """d > 256 (streamed query tile): CTA pairs (even tile counts), AR8 (q <= 8), helper
    producer warps (<= 96 queries in a tile), the block finalize and the histogram threshold
    (q < 148, k' >= 64) -- each with every row delivery."""
    rng = np.random.default_rng(SEED_BASE + 5000 + seed)
    n = int(rng.integers(1, 30000))
    d = int(rng.choice([264, 320, 512, 768, 1032, 1536]))
    q = int(rng.choice([1, 5, 8, 9, 33, 96, 97, 129, 200, 256, 257, 384, 512]))
    k = int(rng.choice([1, 10, 50, 100, 150, 240]))
    metric = int(rng.choice([oracle.L2, oracle.IP, oracle.COS]))
    lo = int(rng.integers(0, 1000))
    pred = [] if rng.integers(0, 4) == 0 else [(0, lo, int(rng.integers(lo - 3, 1000)))]
    rows = [None, 1, 2][int(rng.integers(0, 3))]
    off = int(rng.integers(0, 1 << 20))
    return rng, n, d, q, k, metric, pred, rows, off


@pytest.mark.parametrize("seed", range(N_CASES_LARGE_D))
def test_fuzz_parity_large_d(vrs, seed):
    rng, n, d, q, k, metric, pred, rows, off = _case_large_d(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off)
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=METRICS[metric], path=vrs.PATH_GEMM,
                           rows=rows)
    torch.cuda.synchronize()
    check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric, row_offset=off)
