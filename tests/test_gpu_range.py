"""Parity of vrs_range_search (threshold selection, PAPER.md L354 / L1436; SPEC.md
L144, L178) against the oracle's orc_range: the same ids in the same (ascending)
order, dists exact to fp32 rounding.  Thresholds are placed away from every
score (ties at tau would depend on fp64 summation order)."""
import numpy as np
import pytest
import torch

import oracle
from oracle import COS, IP, L2

pytestmark = pytest.mark.gpu
METRICS = {L2: "l2", IP: "ip", COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _tau_between(scores, rank, metric):
    """A threshold strictly between the rank-th and (rank+1)-th best of `scores`."""
    s = np.sort(scores)[::-1] if metric != L2 else np.sort(scores)
    return float((s[rank] + s[rank + 1]) / 2)


def _check(vrs, X, attrs, pred, Q, tau, metric, rows=None, precision=None):
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], precision=precision)
    off, ids, dists = ix.range_search(torch.from_numpy(Q).cuda(), pred, tau=tau, metric=METRICS[metric], rows=rows,
                                      capacity=4)
    torch.cuda.synchronize()
    roff, rids, rd, _ = oracle.range_search(X, attrs, pred, Q, tau, metric)
    assert off.cpu().numpy().tolist() == roff.tolist()
    assert ids.cpu().numpy().tolist() == rids.tolist()
    assert np.allclose(dists.cpu().numpy(), rd, rtol=1e-6, atol=1e-7)
    return len(rids)


CASES = [
    # n, d, q, metric, pred, rank of tau within the first query's qualifying scores
    (3000, 128, 5, IP, [(0, 0, 499)], 40),
    (5000, 64, 3, L2, [], 25),
    (4099, 32, 130, COS, [(0, 100, 899)], 60),
    (20000, 256, 7, IP, [(0, 0, 9)], 5),        # ~1 % selectivity
    (2000, 768, 2, L2, [(0, 0, 699)], 30),
    (4000, 8, 4, IP, [], 50),                    # small d: the bound's rounding terms dominate
    (4000, 16, 4, L2, [(0, 0, 799)], 30),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[0]}-d{c[1]}-q{c[2]}-m{c[3]}")
@pytest.mark.parametrize("rows", [0, 1, 2], ids=["auto", "gather", "masked"])
@pytest.mark.parametrize("prec", [1, 2, 3], ids=["tf32", "bf16", "fp16"])
def test_range_parity(vrs, case, rows, prec):
    n, d, q, metric, pred, rank = case
    rng = np.random.default_rng(n + d + q)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    _, _, sel = oracle.select(attrs, n, pred)
    s0 = oracle.score(X, Q[0], sel, metric)
    tau = _tau_between(s0, rank, metric)
    total = _check(vrs, X, attrs, pred, Q, tau, metric, rows=rows, precision=prec)
    assert total >= rank + 1


def test_range_spec_examples(vrs):
    """SPEC.md L156 / L158 (rows padded to d = 4 with zeros: the scores are unchanged)."""
    rows = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0.8, 0.6, 0, 0]], dtype=np.float32)
    q = np.array([[1, 0, 0, 0]], dtype=np.float32)
    attrs = [np.array([0, 0, 1], dtype=np.int32)]
    ix = vrs.Index(torch.from_numpy(rows).cuda(), [torch.from_numpy(attrs[0]).cuda()])
    off, ids, dists = ix.range_search(torch.from_numpy(q).cuda(), [], tau=0.9, metric="cos")
    assert ids.cpu().tolist() == [0] and np.allclose(dists.cpu().numpy(), [1.0])
    off, ids, dists = ix.range_search(torch.from_numpy(q).cuda(), [(0, 1, 1)], tau=0.5, metric="cos")
    assert ids.cpu().tolist() == [2] and np.allclose(dists.cpu().numpy(), [0.8])


def test_range_extremes_and_errors(vrs):
    rng = np.random.default_rng(5)
    n, d = 1500, 64
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 10, n).astype(np.int32)]
    Q = rng.standard_normal((3, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(attrs[0]).cuda()])
    Qd = torch.from_numpy(Q).cuda()
    _, _, sel = oracle.select(attrs, n, [(0, 2, 4)])
    off, ids, _ = ix.range_search(Qd, [(0, 2, 4)], tau=-np.inf, metric="ip")      # every qualifying row
    assert off.cpu().tolist() == [0, len(sel), 2 * len(sel), 3 * len(sel)]
    assert ids[: len(sel)].cpu().tolist() == sel.tolist()
    off, ids, _ = ix.range_search(Qd, [(0, 5, 4)], tau=-np.inf, metric="ip")       # empty selection
    assert off.cpu().tolist() == [0, 0, 0, 0] and ids.numel() == 0
    off, ids, _ = ix.range_search(Qd[:0], [], tau=0.0, metric="l2")                 # q = 0
    assert off.cpu().tolist() == [0]
    Qz = torch.zeros(1, d, device="cuda")                                           # zero COS query
    off, ids, _ = ix.range_search(Qz, [], tau=-1.0, metric="cos")
    assert off.cpu().tolist() == [0, 0]
    with pytest.raises(vrs.VrsError):
        ix.range_search(Qd, [], tau=float("nan"), metric="ip")
