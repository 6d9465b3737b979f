"""GPU parity: libvrs (through the C ABI) vs the CPU oracle on seeded inputs.

Sizes span several tiles and ragged tails; selectivities include 0, tiny,
partial and 1; every metric and both distance paths.  Acceptance rules in
tests/parity.py."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from parity import check_select, check_topk

pytestmark = pytest.mark.gpu

I32MIN, I32MAX = -(2 ** 31), 2 ** 31 - 1
METRICS = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}


@pytest.fixture(scope="module")
def vrs():
    import paper_2403_15807_b200 as m
    m.library()
    return m


def _data(n, d, seed=0, mod=1000, nattr=1, kind="gauss"):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    if kind == "norm":
        X /= np.linalg.norm(X, axis=1, keepdims=True)
    attrs = [rng.integers(0, mod, n).astype(np.int32)]
    if nattr > 1:
        attrs.append(rng.integers(0, 64, n).astype(np.uint8))
    return X, attrs


def _run(vrs, X, attrs, pred, Q, k, metric, path=None, rows=None, off=0):
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off)
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=METRICS[metric], path=path, rows=rows)
    torch.cuda.synchronize()
    return ids.cpu().numpy(), dists.cpu().numpy()


# ------------------------------------------------------------------ selection

@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 1024, 1025, 10007, 250_001])
def test_select_bit_exact(vrs, n):
    X, attrs = _data(n, 4, seed=n, nattr=2)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    for pred in ([], [(0, I32MIN, 99)], [(0, 500, 499)], [(0, 100, 899), (1, 3, 40)], [(1, 0, 255)],
                 [(0, -5, 10 ** 12)], [(0, 0, 0)], [(1, 200, 300)]):
        bm, cnt, ids = ix.select(pred, with_ids=True)
        torch.cuda.synchronize()
        check_select(bm, cnt, ids, attrs, n, pred)


def test_select_errors(vrs):
    X, attrs = _data(100, 4)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    with pytest.raises(vrs.VrsError) as e:
        ix.select([(3, 0, 1)])
    assert e.value.status == 2    # ENOTFOUND


# ------------------------------------------------------------------ search parity

CASES = [
    # n, d, q, k, metric, pred
    (1, 8, 1, 1, oracle.L2, []),
    (33, 8, 3, 5, oracle.IP, [(0, 0, 499)]),
    (1000, 1, 2, 10, oracle.L2, []),
    (1000, 127, 7, 10, oracle.IP, [(0, I32MIN, 99)]),
    (4099, 128, 8, 10, oracle.L2, [(0, I32MIN, 99)]),
    (4099, 128, 16, 64, oracle.COS, [(0, 0, 499)]),
    (10007, 256, 1, 100, oracle.IP, []),
    (10007, 256, 5, 240, oracle.L2, [(0, 0, 899)]),
    (5000, 1027, 3, 10, oracle.COS, [(0, 0, 599)]),
    (20000, 768, 2, 100, oracle.L2, [(0, I32MIN, 9)]),     # ~1 % selectivity
    (20000, 64, 33, 50, oracle.IP, [(0, 0, 999)]),
    (3000, 128, 9, 10, oracle.L2, [(0, 5000, 6000)]),      # selectivity 0 -> padding
    (300, 128, 4, 240, oracle.IP, [(0, 0, 99)]),           # k > N_sel -> padding
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[0]}-d{c[1]}-q{c[2]}-k{c[3]}-m{c[4]}")
@pytest.mark.parametrize("path", [None, 1], ids=["auto", "scan"])
def test_search_parity(vrs, case, path):
    n, d, q, k, metric, pred = case
    X, attrs = _data(n, d, seed=n + d, kind="norm" if metric == oracle.IP and d == 128 else "gauss")
    Q = np.random.default_rng(q).standard_normal((q, d)).astype(np.float32)
    gi, gd = _run(vrs, X, attrs, pred, Q, k, metric, path=path)
    check_topk(gi, gd, X, attrs, pred, Q, k, metric)


def test_row_offset_and_determinism(vrs):
    X, attrs = _data(5000, 64, seed=3)
    Q = np.random.default_rng(1).standard_normal((4, 64)).astype(np.float32)
    pred = [(0, 0, 299)]
    off = 123_456_789
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], row_offset=off)
    Qd = torch.from_numpy(Q).cuda()
    a = ix.search(Qd, pred, k=20, metric="l2")
    b = ix.search(Qd, pred, k=20, metric="l2")
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])      # bit-identical repeats
    check_topk(a[0].cpu().numpy(), a[1].cpu().numpy(), X, attrs, pred, Q, 20, oracle.L2, row_offset=off)


def test_identical_vector_distance_zero(vrs):
    X, attrs = _data(2000, 32, seed=5)
    Q = X[[17, 1999, 0]].copy()
    gi, gd = _run(vrs, X, attrs, [], Q, 3, oracle.L2)
    assert gi[:, 0].tolist() == [17, 1999, 0] and (gd[:, 0] == 0).all()


def test_q_zero_and_errors(vrs):
    X, attrs = _data(100, 16)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    Qd = torch.zeros(2, 16, device="cuda")
    ids, _ = ix.search(torch.zeros(0, 16, device="cuda"), [], k=5)     # q = 0: no-op
    assert ids.shape == (0, 5)
    cases = [
        (dict(k=0), 1), (dict(k=241), 7), (dict(metric=9), 1), (dict(pred=[(1, 0, 1)]), 2),
        (dict(pred=[(0, 0, 1)] * 9), 7),
    ]
    for kw, status in cases:
        args = dict(pred=[], k=5, metric="l2")
        args.update(kw)
        with pytest.raises(vrs.VrsError) as e:
            ix.search(Qd, **args)
        assert e.value.status == status, kw
    # the binding validates tensors before the call ...
    for bad in (torch.zeros(2, 16), torch.zeros(2, 8, device="cuda"), torch.zeros(2, 16, device="cuda").double(),
                torch.zeros(16, 2, device="cuda").t()):
        with pytest.raises(ValueError):
            ix.search(bad, [], k=5)
    with pytest.raises(ValueError):                          # wrong out shape / dtype
        ix.search(Qd, [], k=5, out=(torch.empty(2, 4, dtype=torch.int64, device="cuda"),
                                    torch.empty(2, 5, device="cuda")))
    # ... and the C ABI itself still rejects a host pointer and a d mismatch (EINVAL)
    import ctypes
    from paper_2403_15807_b200 import _lib
    lib = vrs.library()
    pr, keep = _lib.make_predicate([])
    out_i = torch.empty(2, 5, dtype=torch.int64, device="cuda")
    out_d = torch.empty(2, 5, device="cuda")
    host_q = torch.zeros(2, 16)
    for qptr, dd in ((host_q.data_ptr(), 16), (Qd.data_ptr(), 8)):
        st = lib.vrs_search_ex(ix._h, ctypes.c_void_p(qptr), 2, dd, ctypes.byref(pr), 5, 0,
                               ctypes.c_void_p(out_i.data_ptr()), ctypes.c_void_p(out_d.data_ptr()), None, None)
        assert st == 1
    Z = X.copy()
    Z[3] = 0
    iz = vrs.Index(torch.from_numpy(Z).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    with pytest.raises(vrs.VrsError) as e:
        iz.search(Qd + 1, [], k=5, metric="cos")
    assert e.value.status == 3                              # EDEGENERATE
    ids, d = ix.search(Qd, [], k=5, metric="cos")           # zero COSINE query -> padding
    assert (ids == -1).all()


def test_merge_matches_oracle(vrs):
    rng = np.random.default_rng(12)
    n, d, k, q = 6000, 48, 25, 6
    X, attrs = _data(n, d, seed=12)
    Q = rng.standard_normal((q, d)).astype(np.float32)
    pred = [(0, 0, 699)]
    cuts = [0, 1500, 3001, 4700, 6000]
    for metric in (oracle.L2, oracle.IP, oracle.COS):
        parts = []
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            parts.append(_run(vrs, X[r0:r1].copy(), [a[r0:r1].copy() for a in attrs], pred, Q, k, metric, off=r0))
        ci = torch.from_numpy(np.stack([p[0] for p in parts])).cuda()
        cd = torch.from_numpy(np.stack([p[1] for p in parts])).cuda()
        mi, md = vrs.merge(ci, cd, k, METRICS[metric])
        torch.cuda.synchronize()
        oi, od = oracle.merge(ci.cpu().numpy(), cd.cpu().numpy(), k, metric)
        assert (mi.cpu().numpy() == oi).all() and (md.cpu().numpy() == od).all()
        check_topk(mi.cpu().numpy(), md.cpu().numpy(), X, attrs, pred, Q, k, metric)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_shaped_reduced(vrs, name):
    """Each BASELINE config's distributions / predicate structure at a size the oracle finishes in seconds."""
    cfg = datagen.CONFIGS[name]
    n = {"c1": cfg.n, "c2": 60_000, "c3": 20_000, "c4": 8_000, "c5": 30_000}[name]
    X, attrs = datagen.corpus(cfg, 0, n, "cpu", n=n)
    Xn, an = X.numpy(), [a.numpy() for a in attrs]
    for sel in cfg.sels:
        pred = datagen.predicate(cfg, sel)
        for q in cfg.qs:
            qq = min(q, 64)
            Q = datagen.queries(cfg, qq, "cpu").numpy()
            gi, gd = _run(vrs, Xn, an, pred, Q, cfg.k, cfg.metric)
            check_topk(gi, gd, Xn, an, pred, Q, cfg.k, cfg.metric)


def test_search_host_end_to_end(vrs):
    X, attrs = _data(3000, 64, seed=9)
    Q = np.random.default_rng(2).standard_normal((5, 64)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    ids, dists = ix.search_host(torch.from_numpy(Q).pin_memory(), [(0, 0, 499)], k=7, metric="ip")
    check_topk(ids.numpy(), dists.numpy(), X, attrs, [(0, 0, 499)], Q, 7, oracle.IP)
    # host_async: several calls enqueued back to back, one synchronisation
    outs = []
    for lo in (0, 100, 200):
        outs.append(ix.search_host(torch.from_numpy(Q).pin_memory(), [(0, lo, lo + 399)], k=7, metric="ip",
                                   host_async=True))
    torch.cuda.synchronize()
    for lo, (i2, d2) in zip((0, 100, 200), outs):
        check_topk(i2.numpy(), d2.numpy(), X, attrs, [(0, lo, lo + 399)], Q, 7, oracle.IP)
    # host_async = 2 (overlap): the stream is not ordered after the downloads; host_fence
    # on a separate stream + its synchronisation completes the results
    outs = []
    for lo in (0, 100, 200, 300):
        outs.append(ix.search_host(torch.from_numpy(Q).pin_memory(), [(0, lo, lo + 399)], k=7, metric="ip",
                                   host_async=2))
    s2 = torch.cuda.Stream()
    ix.host_fence(s2)
    s2.synchronize()
    for lo, (i2, d2) in zip((0, 100, 200, 300), outs):
        check_topk(i2.numpy(), d2.numpy(), X, attrs, [(0, lo, lo + 399)], Q, 7, oracle.IP)


@pytest.mark.parametrize("dups", [3, 200], ids=["few-dups", "many-dups"])
@pytest.mark.parametrize("k", [10, 100], ids=["k10", "k100"])
def test_exact_ties_go_to_lower_ids(vrs, dups, k):
    """Duplicated rows score identically: the returned ids must be the oracle's
    (lowest ids among the tied rows), through every selection stage (probe
    threshold, list buffers, finalize's bucket / radix selection)."""
    rng = np.random.default_rng(dups + k)
    n, d = 30000, 128
    X = rng.standard_normal((n, d)).astype(np.float32)
    src = rng.integers(0, n, 40)
    for s in src:   # `dups` copies of 40 rows scattered over the corpus
        X[rng.integers(0, n, dups)] = X[s]
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = X[src[:6]] + 1e-3 * rng.standard_normal((6, d)).astype(np.float32)
    for metric in (oracle.L2, oracle.IP):
        gi, gd = _run(vrs, X, attrs, [(0, 0, 899)], Q, k, metric)
        ri, rd, _ = oracle.search(X, attrs, [(0, 0, 899)], Q, k, metric)
        assert (gi == ri).all()
        assert np.allclose(gd, rd, rtol=1e-6)


@pytest.mark.parametrize("k", [10, 100], ids=["k10", "k100"])
def test_exact_ties_crowd(vrs, k):
    """One row duplicated 3000 times and queried by itself (q <= 2: the small-batch block
    finalize): thousands of candidates share the k'-th key, so the selection resolves
    them by id (one-valued key range / more ties than the tie buffer)."""
    rng = np.random.default_rng(7 + k)
    n, d = 20000, 64
    X = rng.standard_normal((n, d)).astype(np.float32)
    X[rng.choice(n, 3000, replace=False)] = X[5]
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = np.stack([X[5], X[5] + 1e-3 * rng.standard_normal(d).astype(np.float32)])
    for metric in (oracle.L2, oracle.IP):
        gi, gd = _run(vrs, X, attrs, [(0, 0, 949)], Q, k, metric)
        ri, rd, _ = oracle.search(X, attrs, [(0, 0, 949)], Q, k, metric)
        assert (gi == ri).all()
        assert np.allclose(gd, rd, rtol=1e-6, atol=1e-30)


def test_binding_rejects_bad_columns(vrs):
    """a short / misplaced attribute column would be read out of bounds by
    select_count_kernel -- the binding refuses it before vrs_load."""
    X = torch.zeros(100, 8, device="cuda")
    for bad in ([torch.zeros(99, dtype=torch.int32, device="cuda")],
                [torch.zeros(100, dtype=torch.int32)],
                [torch.zeros(100, 2, dtype=torch.int32, device="cuda")]):
        with pytest.raises(ValueError):
            vrs.Index(X, bad)
    with pytest.raises(ValueError):
        vrs.Index(X.double(), [])


_SELECT_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2403_15807_b200 as vrs
from parity import check_select
for n in (1, 8193, 250_001, 1_000_003):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 4)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32), rng.integers(0, 64, n).astype(np.uint8)]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    for pred in ([], [(0, -5, 99)], [(0, 500, 499)], [(0, 100, 899), (1, 3, 40)]):
        bm, cnt, ids = ix.select(pred, with_ids=True)
        torch.cuda.synchronize()
        check_select(bm, cnt, ids, attrs, n, pred)
print("OK")
'''


def test_select_prefix_kernel(vrs):
    """The chunk-prefix kernel large corpora use (> 4096 chunks of 8192 rows), forced for
    every size by VRS_SELECT_DIRECT_MAX=0 (read once per process: a subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VRS_SELECT_DIRECT_MAX="0")
    r = subprocess.run([sys.executable, "-c", _SELECT_SCRIPT, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]


def test_select_large_corpus(vrs):
    """n = 40M rows (4883 chunks > 4096): the chunk prefix by select_prefix_kernel."""
    n = 40_000_000
    rng = np.random.default_rng(11)
    X = torch.randn((n, 4), dtype=torch.float32, device="cuda")
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    ix = vrs.Index(X, [torch.from_numpy(attrs[0]).cuda()])
    for pred in ([(0, 0, 9)], [(0, 0, 499)]):
        bm, cnt, ids = ix.select(pred, with_ids=True)
        torch.cuda.synchronize()
        check_select(bm, cnt, ids, attrs, n, pred)
