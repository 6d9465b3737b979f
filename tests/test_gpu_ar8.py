"""Small batches with the query tile resident as 8 rows per K block (tc_kernel.cuh AR8:
q <= 8, 16-bit operands, 4 < nk <= 32 K blocks; the MMA reads the 8 rows with stride 0):
parity with the oracle across d (nk 5 .. 32, and 33: the streamed tile), q around the
limit, every metric and row delivery."""
import numpy as np
import pytest
import torch

import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu
M = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


@pytest.mark.parametrize("d", [264, 768, 1536, 2048, 2056])
@pytest.mark.parametrize("q", [1, 5, 8, 9])
def test_ar8_parity(vrs, d, q):
    rng = np.random.default_rng(d * 10 + q)
    n = 7000
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    for metric, pred, rows, k in ((oracle.IP, [(0, 0, 299)], None, 10), (oracle.L2, [], None, 100),
                                  (oracle.COS, [(0, 100, 899)], vrs.ROWS_MASKED, 30),
                                  (oracle.IP, [(0, 0, 999)], vrs.ROWS_GATHER, 64)):
        ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=M[metric], path=vrs.PATH_GEMM, rows=rows)
        torch.cuda.synchronize()
        check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric)
