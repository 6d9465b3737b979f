"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the default index and search options), on sampled outputs: every cell of
the C2 grid (1M x 128) and of one C5 shard (2.5M x 256, clustered, cosine) runs
its full batch; three queries per cell (first, middle, last) are re-computed by
the oracle over all rows; every selectivity's bitmap and count are compared in
full.  C3 and the C4 shard (test_full_size_exact): every cell, the oracle over the
selection's rows in bounded host chunks."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu
METRICS = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_full_size_sampled(vrs, name):
    cfg = datagen.CONFIGS[name]
    r0, r1, _ = datagen.rows_of(cfg, 1, 0)
    dev = torch.device("cuda", 0)
    X, attrs = datagen.corpus(cfg, r0, r1, dev)
    Qall = datagen.queries(cfg, max(cfg.qs), dev)
    ix = vrs.Index(X, attrs, row_offset=r0)
    Xh, ah = X.cpu().numpy(), [a.cpu().numpy() for a in attrs]
    Qh = Qall.cpu().numpy()
    n = r1 - r0
    for s in cfg.sels:
        pred = datagen.predicate(cfg, s)
        bm, cnt, _ = ix.select(pred)
        obm, ocnt, _ = oracle.select(ah, n, pred)
        assert int(cnt.item()) == ocnt
        assert np.array_equal(bm.cpu().numpy().view(np.uint32), obm[: bm.numel()])
        for q in cfg.qs:
            ids, dists = ix.search(Qall[:q], pred, k=cfg.k, metric=METRICS[cfg.metric])
            torch.cuda.synchronize()
            rows = sorted({0, q // 2, q - 1})
            check_topk(ids.cpu().numpy()[rows], dists.cpu().numpy()[rows], Xh, ah, pred, Qh[rows], cfg.k,
                       cfg.metric, row_offset=r0)



def _oracle_over_selection(X_dev, ah, n, pred, Qs, k, metric, row_offset):
    """The oracle's top-k of Qs over the rows ITS OWN selection keeps, in chunks of 400k
    rows copied to the host (bounded memory) and merged by oracle.merge; chunk positions
    map back through the oracle's ascending ids (the id tie-break is unchanged)."""
    _, cnt, sel = oracle.select(ah, n, pred)
    pad = np.inf if metric == oracle.L2 else -np.inf
    if cnt == 0:
        return np.full((Qs.shape[0], k), -1, np.int64), np.full((Qs.shape[0], k), pad, np.float32)
    parts_i, parts_d = [], []
    for c0 in range(0, cnt, 400_000):
        sl = sel[c0:c0 + 400_000]
        Xs = X_dev.index_select(0, torch.from_numpy(sl).to(X_dev.device)).cpu().numpy()
        li, ld, _ = oracle.search(Xs, [], [], Qs, k, metric, 0)
        parts_i.append(np.where(li >= 0, sl[np.clip(li, 0, None)] + row_offset, -1))
        parts_d.append(ld)
    if len(parts_i) == 1:
        return parts_i[0], parts_d[0]
    return oracle.merge(np.stack(parts_i), np.stack(parts_d), k, metric)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_exact(vrs, name):
    """C3 (10M x 768, L2, k = 100) and one C4 shard (6.25M x 1536, IP, k = 100) at their
    full sizes: every cell of the grid (all selectivities x query counts) in the bench's
    default configuration, three sampled queries per cell (first, middle, last) against
    the oracle over the whole selection (_oracle_over_selection).  Certified exactness:
    ids identical rank for rank, dists within one fp32 ulp of fp32(oracle fp64)."""
    cfg = datagen.CONFIGS[name]
    r0, r1, _ = datagen.rows_of(cfg, 1, 0)
    dev = torch.device("cuda", 0)
    X, attrs = datagen.corpus(cfg, r0, r1, dev)
    Qall = datagen.queries(cfg, max(cfg.qs), dev)
    ix = vrs.Index(X, attrs, row_offset=r0)
    ah = [a.cpu().numpy() for a in attrs]
    Qh = Qall.cpu().numpy()
    n = r1 - r0
    sampled = sorted({r for q in cfg.qs for r in (0, q // 2, q - 1)})
    where = {r: i for i, r in enumerate(sampled)}
    for s in cfg.sels:
        pred = datagen.predicate(cfg, s)
        ri, rd = _oracle_over_selection(X, ah, n, pred, Qh[sampled], cfg.k, cfg.metric, r0)
        for q in cfg.qs:
            ids, dists = ix.search(Qall[:q], pred, k=cfg.k, metric=METRICS[cfg.metric])
            torch.cuda.synchronize()
            rows = sorted({0, q // 2, q - 1})
            gi, gd = ids.cpu().numpy()[rows], dists.cpu().numpy()[rows]
            oi, od = ri[[where[r] for r in rows]], rd[[where[r] for r in rows]]
            assert np.array_equal(gi, oi), f"{name} s={s} q={q}: ids differ from the oracle's"
            fin = np.isfinite(od)
            ulp = np.spacing(np.abs(od).astype(np.float32))
            err = np.abs(gd.astype(np.float64) - od.astype(np.float64))
            assert ((err <= ulp) | ~fin).all() and np.array_equal(np.isfinite(gd), fin), \
                f"{name} s={s} q={q}: dists more than 1 ulp from fp32(oracle fp64)"
