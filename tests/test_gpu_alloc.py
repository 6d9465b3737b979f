"""Memory ownership (SURVEY.md 8(b) "Ownership"): the index's derived
data and every call's scratch come from the caller's allocator -- torch's caching allocator
through the binding by default -- and a NULL from it is VRS_ENOMEM; without an allocator
libvrs's own stream-ordered pool keeps at most 2 GiB of freed scratch."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from parity import check_topk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _data(n=50000, d=128, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((64, d)).astype(np.float32)
    return X, attrs, Q


def test_torch_allocator_no_library_pool(vrs):
    """Default index: searches of every path allocate through torch; libvrs's own pool does not
    grow, and torch's allocated bytes return to the baseline once the results are dropped."""
    X, attrs, Q = _data()
    torch.cuda.synchronize()
    pool0 = vrs.pool_reserved_bytes()
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    Qd = torch.from_numpy(Q).cuda()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    for pred in ([], [(0, 0, 99)], [(0, 0, 699)]):
        for path in (None, vrs.PATH_SCAN):
            ids, dists = ix.search(Qd, pred, k=10, metric="ip", path=path)
            torch.cuda.synchronize()
            check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, 10, oracle.IP)
            del ids, dists
    off, rid, rd = ix.range_search(Qd[:4], [], tau=8.0, metric="ip")
    del off, rid, rd
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == base
    assert vrs.pool_reserved_bytes() == pool0


def _failing_allocator(vrs, limit):
    """An allocator that serves requests up to `limit` bytes through torch and fails larger ones."""
    from paper_2403_15807_b200 import _lib

    def alloc(nbytes, stream, ctx):
        if nbytes > limit:
            return None
        return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)

    def free(ptr, stream, ctx):
        if ptr:
            torch.cuda.caching_allocator_delete(ptr)

    return _lib.Allocator(_lib.ALLOC_FN(alloc), _lib.FREE_FN(free), None)


def test_enomem_mapping(vrs):
    X, attrs, Q = _data(20000, 64)
    Xd = torch.from_numpy(X).cuda()
    A = [torch.from_numpy(a).cuda() for a in attrs]
    with pytest.raises(vrs.VrsError) as e:        # the load's own allocation fails
        vrs.Index(Xd, A, allocator=_failing_allocator(vrs, 1024))
    assert e.value.status == 4
    # enough for the index (norms + shadow), too little for a search's scratch
    need = 20000 * (4 + 4) + 2 * 20000 * 64 * 2 + 4096   # norms + the fp16 shadow's two halves
    ix = vrs.Index(Xd, A, allocator=_failing_allocator(vrs, need))
    with pytest.raises(vrs.VrsError) as e:
        ix.search(torch.from_numpy(Q).cuda(), [], k=10, metric="l2")
    assert e.value.status == 4
    # the index is still usable for calls that fit
    ix2 = vrs.Index(Xd, A, allocator=_failing_allocator(vrs, 1 << 40))
    ids, dists = ix2.search(torch.from_numpy(Q).cuda(), [], k=10, metric="l2")
    torch.cuda.synchronize()
    check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, [], Q, 10, oracle.L2)


def test_library_pool_is_bounded(vrs):
    """allocator=None: a search whose scratch (the gathered selection) exceeds the 2 GiB the
    pool keeps leaves at most 2 GiB reserved after a synchronisation."""
    n, d = 3_000_000, 512
    X = torch.randn(n, d, device="cuda")
    a0 = torch.randint(0, 1000, (n,), dtype=torch.int32, device="cuda")
    ix = vrs.Index(X, [a0], allocator=None, precision=vrs.PREC_TF32)
    Q = torch.randn(2048, d, device="cuda")
    ids, dists = ix.search(Q, [(0, 0, 799)], k=10, metric="ip")   # X_sel of 80 % of 6 GB rows
    torch.cuda.synchronize()
    assert ids.shape == (2048, 10)
    assert 0 <= vrs.pool_reserved_bytes() <= (2 << 30) + (64 << 20)
