"""Parity of the tcgen05 tensor-core path (forced) vs the oracle: TF32 selection
with over-fetch + exact re-score must meet the same acceptance rules."""
import numpy as np
import pytest
import torch

import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu
I32MIN = -(2 ** 31)
METRICS = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _run(vrs, X, attrs, pred, Q, k, metric, off=0, rows=None, precision=None):
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off,
                   precision=precision)
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=METRICS[metric], path=vrs.PATH_GEMM,
                           rows=rows)
    torch.cuda.synchronize()
    assert vrs.last_path() == vrs.PATH_GEMM
    if precision is not None:
        assert vrs.last_precision() == precision
    return ids.cpu().numpy(), dists.cpu().numpy()


GEMM_CASES = [
    # n, d, q, k, metric, pred
    (256, 32, 128, 10, oracle.IP, []),                 # one tile, one K block
    (1000, 128, 1, 10, oracle.L2, []),                 # ragged rows, q = 1 (M padded)
    (4099, 128, 130, 10, oracle.IP, [(0, 0, 99)]),     # two query tiles, ragged, 10 %
    (9000, 64, 300, 64, oracle.COS, [(0, 0, 499)]),
    (5000, 4, 17, 5, oracle.L2, []),                   # d = 4: K block zero-filled
    (3000, 100, 40, 100, oracle.L2, [(0, 0, 899)]),    # d % 32 != 0
    (20000, 256, 64, 240, oracle.IP, [(0, I32MIN, 9)]),   # k = K_MAX, ~1 % selectivity
    (12000, 768, 9, 100, oracle.L2, [(0, 0, 299)]),
    (2000, 128, 16, 10, oracle.IP, [(0, 5000, 6000)]),    # selectivity 0
    # q >= 592: the warp-per-query threshold / finalize kernels, k' <= 64 / <= 128 / > 128
    (6000, 128, 1000, 10, oracle.IP, [(0, 0, 299)]),
    (12000, 64, 700, 50, oracle.COS, [(0, 0, 499)]),
    (8000, 128, 600, 100, oracle.L2, []),
    (5000, 64, 640, 200, oracle.IP, [(0, 0, 799)]),
    (3000, 32, 20000, 10, oracle.L2, [(0, 0, 599)]),   # 157 query tiles, many more CTAs than SMs
]


@pytest.mark.parametrize("case", GEMM_CASES, ids=lambda c: f"n{c[0]}-d{c[1]}-q{c[2]}-k{c[3]}-m{c[4]}")
@pytest.mark.parametrize("rows", [0, 1, 2], ids=["auto", "gather", "masked"])
@pytest.mark.parametrize("prec", [1, 2, 3], ids=["tf32", "bf16", "fp16"])
def test_gemm_parity(vrs, case, rows, prec):
    n, d, q, k, metric, pred = case
    if prec in (2, 3) and d % 8:
        pytest.skip("a 16-bit shadow needs d % 8 == 0")
    rng = np.random.default_rng(n * 7 + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    gi, gd = _run(vrs, X, attrs, pred, Q, k, metric, rows=rows, precision=prec)
    check_topk(gi, gd, X, attrs, pred, Q, k, metric)


def test_gemm_matches_scan_ids(vrs):
    """Both distance engines return the same exact top-k on tie-free data."""
    rng = np.random.default_rng(77)
    n, d, q, k = 30000, 128, 200, 10
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    Qd = torch.from_numpy(Q).cuda()
    a = ix.search(Qd, [(0, 0, 499)], k=k, metric="ip", path=vrs.PATH_GEMM)
    b = ix.search(Qd, [(0, 0, 499)], k=k, metric="ip", path=vrs.PATH_SCAN)
    torch.cuda.synchronize()
    same = (a[0] == b[0]).float().mean().item()
    assert same > 0.999
    assert torch.allclose(a[1], b[1], rtol=1e-6)
