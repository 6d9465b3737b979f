"""Batches beyond 65535 queries (CUDA's grid.y / grid.z limit): every launch that indexes
queries, query tiles or query groups by a grid dimension -- tensor-core pass, FFMA scan,
thresholds, finalize, exact fallback, range mode, merge -- on a small corpus, against the
oracle on the first, last and sampled queries (queries are independent, so the oracle over
the sample is the oracle of the batch)."""
import numpy as np
import pytest
import torch

import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu
Q_BIG = 70_003


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _data(d, n=3001, seed=77):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((Q_BIG, d)).astype(np.float32)
    sample = np.unique(np.concatenate([[0, 1, 127, 128, 65535, 65536, 65537, Q_BIG - 2, Q_BIG - 1],
                                       rng.integers(0, Q_BIG, 40)]))
    return X, attrs, Q, sample


@pytest.mark.parametrize("path,d,k,metric", [("gemm", 64, 10, oracle.IP), ("gemm", 320, 100, oracle.L2),
                                            ("scan", 64, 5, oracle.COS), ("scan", 12, 10, oracle.L2),
                                            (None, 128, 10, oracle.IP)])
def test_topk_above_65535_queries(vrs, path, d, k, metric):
    X, attrs, Q, sample = _data(d)
    pred = [(0, 100, 699)]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    p = {"gemm": vrs.PATH_GEMM, "scan": vrs.PATH_SCAN, None: None}[path]
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=["l2", "ip", "cos"][metric], path=p)
    torch.cuda.synchronize()
    gi, gd = ids.cpu().numpy(), dists.cpu().numpy()
    assert (gi >= 0).all(), "every query has k qualifying rows here"
    check_topk(gi[sample], gd[sample], X, attrs, pred, Q[sample], k, metric)


def test_range_above_65535_queries(vrs):
    X, attrs, Q, sample = _data(64)
    pred = [(0, 0, 499)]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    tau = 20.0   # IP of N(0,1)^64 pairs: sd 8 -> ~0.6 % of the ~1500 qualifying rows per query
    o, ids, dists = ix.range_search(torch.from_numpy(Q).cuda(), pred, tau=tau, metric="ip")
    torch.cuda.synchronize()
    o, ids = o.cpu().numpy(), ids.cpu().numpy()
    assert o.shape[0] == Q_BIG + 1 and o[-1] == ids.shape[0]
    for j in sample:
        ro, rids, _, _ = oracle.range_search(X, attrs, pred, Q[j:j + 1], tau, oracle.IP)
        assert ids[o[j]:o[j + 1]].tolist() == rids.tolist(), j


def test_merge_above_65535_queries(vrs):
    rng = np.random.default_rng(5)
    parts, k = 3, 8
    d = np.sort(rng.standard_normal((parts, Q_BIG, k)).astype(np.float32), axis=2)   # L2: ascending
    i = rng.permutation(parts * Q_BIG * k).reshape(parts, Q_BIG, k).astype(np.int64)
    gi, gd = vrs.merge(torch.from_numpy(i).cuda(), torch.from_numpy(d).cuda(), k, "l2")
    torch.cuda.synchronize()
    ri, rd = oracle.merge(i, d, k, oracle.L2)
    assert (gi.cpu().numpy() == ri).all() and (gd.cpu().numpy() == rd).all()
