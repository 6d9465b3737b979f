"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the default index and search options), on sampled outputs: every cell of
the C2 grid (1M x 128) and of one C5 shard (2.5M x 256, clustered, cosine) runs
its full batch; three queries per cell (first, middle, last) are re-computed by
the oracle over all rows; every selectivity's bitmap and count are compared in
full.  (C3 / C4 shards need 30-40 GB host copies for the oracle: their reduced
shapes are in test_gpu_parity.py, their full sizes in bench.py's sampled check.)"""
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
