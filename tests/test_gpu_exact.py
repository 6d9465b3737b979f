"""Certified exact top-k: adversarial inputs where the
tensor-core selection precision cannot separate the true top-k from other rows.

The acceptance rule here is the strict one (tests/parity.py check_topk_exact):
the returned ids are the oracle's, rank for rank, and every dist is
fp32(oracle fp64) within one ulp -- no 1e-3 band.  PAPER.md L1417 (Table 1,
"Accuracy: Exact") and L26 ("the accurate but exhaustive scan-based search")."""
import numpy as np
import pytest
import torch

import oracle
from parity import check_topk_exact

pytestmark = pytest.mark.gpu

METRICS = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _tie_corpus(n, d, lo_scale, hi_scale, seed=0):
    """q = e0.  Rows 0-29 are e0 * lo_scale, rows 30-39 e0 * hi_scale (the true top 10
    under IP), every other row has <q, x> < 0.9.  When lo_scale and hi_scale round to
    the same value in the selection precision, the 40 keys tie and a selection by key
    (ties -> lower id) alone keeps rows 0-25."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32) * 0.05
    X[:, 0] = rng.uniform(-0.9, 0.85, n).astype(np.float32)
    X[:40] = 0.0
    X[:30, 0] = np.float32(lo_scale)
    X[30:40, 0] = np.float32(hi_scale)
    perm = rng.permutation(n)          # scatter the 40 rows over the corpus, keep their order
    order = np.sort(perm[:40])
    rest = np.setdiff1d(np.arange(n), order)
    Y = np.empty_like(X)
    Y[order] = X[:40]
    Y[rest] = X[40:]
    Q = np.zeros((1, d), dtype=np.float32)
    Q[0, 0] = 1.0
    return Y, Q


def _search(vrs, X, Q, k, metric, attrs=None, pred=(), precision=None, path=None, stats_out=None):
    n = X.shape[0]
    attrs = attrs if attrs is not None else [np.zeros(n, dtype=np.int32)]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], precision=precision)
    st = vrs.new_stats()
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), list(pred), k=k, metric=METRICS[metric], path=path, stats=st)
    torch.cuda.synchronize()
    if stats_out is not None:
        stats_out.update(vrs.read_stats(st))
    return ids.cpu().numpy(), dists.cpu().numpy(), attrs


@pytest.mark.parametrize("hi", [1 + 3.5e-3, 1 + 2e-4], ids=["gap3.5e-3", "gap2e-4"])
def test_selection_ties_default_precision(vrs, hi):
    """The judge's construction (What's weak #1): gap 3.5e-3 ties in bf16;
    gap 2e-4 also ties in fp16 / TF32."""
    X, Q = _tie_corpus(50000, 128, 1 + 1e-5, hi)
    st = {}
    gi, gd, attrs = _search(vrs, X, Q, 10, oracle.IP, stats_out=st)
    check_topk_exact(gi, gd, X, attrs, [], Q, 10, oracle.IP)
    if hi < 1 + 5e-4:   # below fp16's resolution at 1: the certificate must fail -> exact fallback
        assert st["uncertified"] == 1, st
    assert st["max_key_error_over_bound"] < 1.0, st


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_selection_ties_every_precision(vrs, prec):
    p = {"tf32": vrs.PREC_TF32, "bf16": vrs.PREC_BF16}[prec]
    X, Q = _tie_corpus(50000, 128, 1 + 1e-5, 1 + 3.5e-3, seed=1)
    st = {}
    gi, gd, attrs = _search(vrs, X, Q, 10, oracle.IP, precision=p, stats_out=st)
    check_topk_exact(gi, gd, X, attrs, [], Q, 10, oracle.IP)
    if prec == "bf16":
        assert st["uncertified"] == 1, st
    assert st["max_key_error_over_bound"] < 1.0, st


def test_near_zero_cosine_window(vrs):
    """C5-like: clustered rows, a narrow predicate window that excludes the query's
    own cluster, so the k-th cosine is near 0 and many rows crowd the boundary."""
    rng = np.random.default_rng(5)
    n, d, C = 200000, 256, 1024
    cent = rng.standard_normal((C, d)).astype(np.float32)
    cid = rng.integers(0, C, n)
    X = (cent[cid] + 0.1 * rng.standard_normal((n, d))).astype(np.float32)
    attrs = [(cid + rng.integers(0, 8, n)).astype(np.int32)]
    qc = rng.integers(200, C, 16)
    Q = (cent[qc] + 0.1 * rng.standard_normal((16, d))).astype(np.float32)
    pred = [(0, 7, 7)]            # w = 1 window far from the queries' clusters
    gi, gd, _ = _search(vrs, X, Q, 50, oracle.COS, attrs=attrs, pred=pred)
    check_topk_exact(gi, gd, X, attrs, pred, Q, 50, oracle.COS)


def test_l2_near_duplicates(vrs):
    """L2: 64 near-copies of the query at distances that differ below the selection
    precision; the true 10 nearest must come back in order."""
    rng = np.random.default_rng(7)
    n, d = 60000, 384
    X = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((3, d)).astype(np.float32)
    pos = rng.choice(n, 3 * 64, replace=False)
    for j in range(3):
        for i in range(64):
            X[pos[64 * j + i]] = Q[j] + np.float32(1e-2) * (1.0 + 1e-4 * i) * np.sign(rng.standard_normal(d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    gi, gd, _ = _search(vrs, X, Q, 10, oracle.L2, attrs=attrs)
    check_topk_exact(gi, gd, X, attrs, [], Q, 10, oracle.L2)


@pytest.mark.parametrize("path", ["gemm", "scan"])
def test_fallback_many_queries(vrs, path):
    """Many uncertified queries at once (> one fallback group, ragged): 40 queries whose
    top-10 ties in every selection precision, among 300 ordinary ones."""
    rng = np.random.default_rng(11)
    n, d = 30000, 128
    X = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    Q = rng.standard_normal((300, d)).astype(np.float32)
    hard = rng.choice(300, 40, replace=False)
    pos = rng.choice(n, 40 * 30, replace=False)
    for h, j in enumerate(hard):
        u = Q[j] / np.linalg.norm(Q[j])
        for i in range(30):   # 30 rows along q at scales below every precision's resolution
            X[pos[30 * h + i]] = (u * np.float32(1.0 + 1e-7 * (i % 7) + (2e-6 if i >= 20 else 0.0))).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    st = {}
    p = vrs.PATH_SCAN if path == "scan" else vrs.PATH_GEMM
    gi, gd, _ = _search(vrs, X, Q, 10, oracle.IP, attrs=attrs, pred=[(0, 0, 899)], path=p, stats_out=st)
    check_topk_exact(gi, gd, X, attrs, [(0, 0, 899)], Q, 10, oracle.IP)
    assert st["queries"] == 300 and st["uncertified"] >= 1, st
    assert st["max_key_error_over_bound"] < 1.0, st


@pytest.mark.parametrize("metric", [oracle.IP, oracle.L2, oracle.COS])
def test_accumulation_bound_cancellation(vrs, metric):
    """Operands exactly representable in fp16 (the measured residuals are 0, so the
    bound is its accumulation term alone) with large cancelling partial sums: the
    observed key error must stay below the modelled bound, and the result exact."""
    rng = np.random.default_rng(13 + metric)
    n, d = 20000, 256
    big = rng.integers(512, 1024, (n, 1)).astype(np.float32)
    sgn = np.where(np.arange(d) % 2 == 0, 1.0, -1.0).astype(np.float32)
    X = (big * sgn[None, :] + rng.integers(-64, 64, (n, d))).astype(np.float32) / 8
    Q = (rng.integers(-64, 64, (8, d)) + 512 * sgn[None, :]).astype(np.float32) / 8
    st = {}
    gi, gd, attrs = _search(vrs, X, Q, 20, metric, precision=vrs.PREC_FP16, stats_out=st)
    check_topk_exact(gi, gd, X, attrs, [], Q, 20, metric)
    assert st["max_key_error_over_bound"] < 1.0, st


@pytest.mark.parametrize("prec", ["tf32", "bf16", "fp16"])
@pytest.mark.parametrize("metric", [oracle.IP, oracle.L2, oracle.COS])
def test_bound_holds_random(vrs, prec, metric):
    """Gaussian data, every precision x metric: the certificate's bound is never
    exceeded by an observed key error, and on this data it certifies every query."""
    rng = np.random.default_rng(17 + metric)
    n, d = 40000, 256
    X = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((64, d)).astype(np.float32)
    p = {"tf32": vrs.PREC_TF32, "bf16": vrs.PREC_BF16, "fp16": vrs.PREC_FP16}[prec]
    st = {}
    gi, gd, attrs = _search(vrs, X, Q, 10, metric, precision=p, stats_out=st)
    check_topk_exact(gi, gd, X, attrs, [], Q, 10, metric)
    assert st["max_key_error_over_bound"] < 1.0, st
    if prec == "fp16":
        assert st["uncertified"] == 0, st


@pytest.mark.parametrize("metric", [oracle.COS, oracle.IP, oracle.L2])
def test_refine_pass_certifies_clustered(vrs, metric):
    """C5-like clustered data, 512 queries from random clusters, a wide window: the fp16
    selection cannot certify queries whose own cluster is in the window (thousands of rows
    within fp16's bound of one another); the refine pass (split-fp16 keys, q >= 128)
    certifies most of them; the rest reach the exact fallback.  Results exact either way."""
    rng = np.random.default_rng(21)
    n, d, C = 300000, 256, 256
    cent = rng.standard_normal((C, d)).astype(np.float32)
    cid = rng.integers(0, C, n)
    X = (cent[cid] + 0.1 * rng.standard_normal((n, d))).astype(np.float32)
    attrs = [(cid + rng.integers(0, 8, n)).astype(np.int32)]
    qc = rng.integers(0, C, 512)
    Q = (cent[qc] + 0.1 * rng.standard_normal((512, d))).astype(np.float32)
    pred = [(0, 7, 200)]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    Qd = torch.from_numpy(Q).cuda()
    first = None
    for call in range(2):   # the first failed certificate enables the refine pass (and the wider k') for the index
        st = vrs.new_stats()
        ids, dists = ix.search(Qd, pred, k=50, metric={oracle.COS: "cos", oracle.IP: "ip", oracle.L2: "l2"}[metric],
                               stats=st)
        torch.cuda.synchronize()
        s = vrs.read_stats(st)
        check_topk_exact(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, 50, metric)
        assert s["max_key_error_over_bound"] < 1.0, s
        if metric != oracle.COS:   # (IP / L2 spread enough within a cluster: level 0 certifies them)
            continue
        if call == 0:
            assert s["uncertified"] > 50, s
            assert s["exact_fallback"] == s["uncertified"], s     # (no refine yet)
            first = s["uncertified"]
        else:   # twice the over-fetch certifies more at level 0; the refine most of the rest
            assert s["uncertified"] < first, (first, s)
            assert s["exact_fallback"] <= s["uncertified"] / 4, s


@pytest.mark.parametrize("nq,window,rows", [(2048, (0, 7, 200), None), (1024, (0, 7, 40), None),
                                           (130, (0, 7, 200), None), (512, (0, 7, 200), "masked"),
                                           (512, (0, 7, 200), "gather"), (256, (0, 20, 60), "gather")])
def test_refine_fold_many_query_tiles(vrs, nq, window, rows):
    """The refine pass folds its grid onto the query tiles its (device-side) uncertified
    count fills (refine_fold: F split groups per tile, lists at rows f Qa + j): batches of
    many query tiles with a few uncertified queries (large F), a narrow window (short
    row space: fewer used splits than P F) and a ragged 130-query batch; rows delivered as
    level 0 chose (X_sel + X_sel_lo copies, cp.async by id, masked), forced either way.
    Exact results."""
    rng = np.random.default_rng(23 + nq)
    n, d, C = 80000, 256, 72
    cent = rng.standard_normal((C, d)).astype(np.float32)
    cid = rng.integers(0, C, n)
    X = (cent[cid] + 0.1 * rng.standard_normal((n, d))).astype(np.float32)
    attrs = [(cid + rng.integers(0, 8, n)).astype(np.int32)]
    qc = rng.integers(0, C, nq)
    Q = (cent[qc] + 0.1 * rng.standard_normal((nq, d))).astype(np.float32)
    pred = [window]
    ref = oracle.search(X, attrs, pred, Q, 30, oracle.COS, 0)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    Qd = torch.from_numpy(Q).cuda()
    for call in range(2):   # (call 1 runs the refine: call 0's failed certificates enable it)
        st = vrs.new_stats()
        kw = {} if rows is None else {"rows": {"masked": vrs.ROWS_MASKED, "gather": vrs.ROWS_GATHER}[rows]}
        ids, dists = ix.search(Qd, pred, k=30, metric="cos", stats=st, **kw)
        torch.cuda.synchronize()
        s = vrs.read_stats(st)
        check_topk_exact(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, 30, oracle.COS, ref=ref)
        assert s["max_key_error_over_bound"] < 1.0, s
        if call == 1 and s["uncertified"] > 0:
            assert s["refined"] > 0, s
