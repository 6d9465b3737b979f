"""Pins for the CPU oracle (oracle/vrs_oracle.c) -- runs without a GPU.

The paper prints no result values, so every pin is
against something other than the oracle itself: closed forms, the SPEC.md
worked examples (tests/golden/spec_examples.json, each cited), invariants of
the definition, and brute force over tiny inputs.
Each pin is chosen so a plausible slip (dropped term, wrong sign / index,
transposed operand, wrong order or tie rule) fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import COS, IP, L2

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
I32MIN, I32MAX = -(2 ** 31), 2 ** 31 - 1


# ----------------------------------------------------------------- predicate

@pytest.mark.parametrize("ex", GOLD["evaluate_predicate"], ids=lambda e: e["cite"][:24])
def test_spec_predicate_examples(ex):
    a = np.array(ex["values"], dtype=np.int32)
    bm, cnt, ids = oracle.select([a], len(a), [(0, ex["lo"], ex["hi"])])
    assert ids.tolist() == ex["ids"] and cnt == len(ex["ids"])


def test_bitmap_layout_lsb_first_tail_zero():
    n = 70
    a = np.arange(n, dtype=np.int32)
    bm, cnt, _ = oracle.select([a], n, [])                      # no clause: all rows
    assert cnt == n
    assert bm.tolist() == [0xFFFFFFFF, 0xFFFFFFFF, 0x3F]       # 70 = 64 + 6 bits, tail zero
    bm, cnt, _ = oracle.select([a], n, [(0, 33, 33)])         # exactly row 33 -> word 1 bit 1
    assert bm.tolist() == [0, 2, 0] and cnt == 1
    bm, cnt, _ = oracle.select([a], n, [(0, 5, 4)])           # lo > hi: selectivity 0
    assert cnt == 0 and not bm.any()


def test_predicate_exhaustive_interval_closed_form():
    """Sum over every interval [lo,hi] of a small domain of the count equals
    sum_i (#intervals containing a_i) = sum_i (a_i-L+1)(H-a_i+1)."""
    rng = np.random.default_rng(7)
    a = rng.integers(0, 6, size=23).astype(np.int32)
    L, H = -1, 6
    total, per_row = 0, np.zeros(len(a), dtype=np.int64)
    for lo in range(L, H + 1):
        for hi in range(lo, H + 1):
            bm, cnt, ids = oracle.select([a], len(a), [(0, lo, hi)])
            total += cnt
            per_row[ids] += 1
            bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[: len(a)]
            assert np.flatnonzero(bits).tolist() == ids.tolist()    # bitmap <-> ids
            assert all(np.diff(ids) > 0)                              # strictly ascending
    expect = (a.astype(np.int64) - L + 1) * (H - a.astype(np.int64) + 1)
    assert per_row.tolist() == expect.tolist()
    assert total == int(expect.sum())


def test_predicate_partition_and_conjunction():
    rng = np.random.default_rng(3)
    n = 1000
    a = rng.integers(0, 100, size=n).astype(np.int32)
    b = rng.integers(0, 64, size=n).astype(np.uint8)
    for t in (0, 17, 50, 99):
        _, c1, i1 = oracle.select([a, b], n, [(0, I32MIN, t)])
        _, c2, i2 = oracle.select([a, b], n, [(0, t + 1, I32MAX)])
        assert c1 + c2 == n and not set(i1) & set(i2)               # complement partitions
    # AND of clauses on different columns == intersection of the single selections
    _, _, ia = oracle.select([a, b], n, [(0, 10, 60)])
    _, _, ib = oracle.select([a, b], n, [(1, 5, 9)])
    _, _, iab = oracle.select([a, b], n, [(0, 10, 60), (1, 5, 9)])
    assert iab.tolist() == sorted(set(ia) & set(ib))
    # two clauses on one column == interval intersection
    _, _, ii = oracle.select([a, b], n, [(0, 10, 60), (0, 40, 80)])
    _, _, ij = oracle.select([a, b], n, [(0, 40, 60)])
    assert ii.tolist() == ij.tolist()
    # uint8 compared as unsigned (255 is large, not -1)
    u = np.array([0, 255, 128], dtype=np.uint8)
    _, _, iu = oracle.select([u], 3, [(0, 200, 300)])
    assert iu.tolist() == [1]


def test_selectivity_binomial_3sigma():
    """realized selectivity within +-3 sigma of the target."""
    import datagen
    cfg = datagen.CONFIGS["c2"]
    n = 200_000
    X, attrs = datagen.corpus(cfg, 0, n, "cpu", n=n, d=4)
    for s in cfg.sels:
        clauses = datagen.predicate(cfg, s)
        p = datagen.expected_selectivity(cfg, clauses)
        _, cnt, _ = oracle.select([attrs[0].numpy()], n, clauses)
        sigma = math.sqrt(n * p * (1 - p))
        assert abs(cnt - n * p) <= 3 * sigma + 1e-9, (s, cnt, n * p)


# ------------------------------------------------------------------- scores

def _score(X, q, metric, ids=None):
    X = np.asarray(X, dtype=np.float32)
    ids = range(len(X)) if ids is None else ids
    return oracle.score(X, np.asarray(q, dtype=np.float32), list(ids), metric)


def test_scores_closed_forms_identical_and_orthogonal():
    x = np.array([1, -2, 3, 4, 0, 5], dtype=np.float32)
    assert _score([x], x, L2)[0] == 0.0                                # identical -> 0
    assert _score([x], x, IP)[0] == float((x.astype(np.int64) ** 2).sum())  # |x|^2 = 55
    assert abs(_score([x], x, COS)[0] - 1.0) < 1e-15                  # identical -> 1
    y = np.array([2, 1, 0, 0, 0, 0], dtype=np.float32)                # x.y = 2 - 2 = 0
    assert _score([y], x, IP)[0] == 0.0 and _score([y], x, COS)[0] == 0.0


def test_scores_worked_integer_examples():
    # L2 squared, direct: [1,2,3] vs [2,2,2] -> 1 + 0 + 1 = 2 (not sqrt(2))
    assert _score([[1, 2, 3]], [2, 2, 2], L2)[0] == 2.0
    # IP sign and orientation: [1,2,3].[-1,0,2] = -1 + 6 = 5
    assert _score([[1, 2, 3]], [-1, 0, 2], IP)[0] == 5.0
    # COS: [3,4] vs [4,-3] orthogonal; [3,4] vs [6,8] parallel; vs e0 -> 3/5
    s = _score([[4, -3], [6, 8], [1, 0]], [3, 4], COS)
    assert s[0] == 0.0 and abs(s[1] - 1.0) < 1e-15 and abs(s[2] - 0.6) < 1e-15


@pytest.mark.parametrize("ex", GOLD["normalize"], ids=lambda e: e["cite"][:24])
def test_spec_normalize_example(ex):
    s = _score([[1, 0], [0, 1]], ex["row"], COS)
    assert abs(s[0] - ex["cos_e0"]) < 1e-15 and abs(s[1] - ex["cos_e1"]) < 1e-15
    assert abs(math.sqrt(_score([ex["row"]], ex["row"], IP)[0]) - ex["norm"]) < 1e-15


@pytest.mark.parametrize("ex", GOLD["similarity_kernel"], ids=lambda e: e["cite"][:24])
def test_spec_similarity_examples(ex):
    assert _score([ex["b"]], ex["a"], IP)[0] == ex["ip"]


def test_scores_basis_and_constant_query_closed_forms():
    rng = np.random.default_rng(11)
    X = rng.integers(-8, 9, size=(7, 13)).astype(np.float32)
    for t in range(13):                                   # basis query e_t: IP = x_t
        e = np.zeros(13, dtype=np.float32)
        e[t] = 1
        assert _score(X, e, IP).tolist() == X[:, t].astype(np.float64).tolist()
    c = 3.0                                               # constant query: expansion closed form
    Xi = X.astype(np.int64)
    expect = (Xi ** 2).sum(1) - 2 * 3 * Xi.sum(1) + 13 * 9
    assert _score(X, np.full(13, c, dtype=np.float32), L2).tolist() == expect.astype(float).tolist()


def test_scores_metric_identities_random():
    """L2 = |q|^2 + |x|^2 - 2 IP  (pins the sign / a dropped term);
    COS = IP / (|q||x|); COS invariant to positive scaling of x; |COS| <= 1."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((50, 37)).astype(np.float32)
    q = rng.standard_normal(37).astype(np.float32)
    l2, ip, cs = _score(X, q, L2), _score(X, q, IP), _score(X, q, COS)
    nq = _score([q], q, IP)[0]
    nx = np.array([_score([x], x, IP)[0] for x in X])
    assert np.allclose(l2, nq + nx - 2 * ip, rtol=1e-12, atol=1e-10)
    assert np.allclose(cs, ip / np.sqrt(nq * nx), rtol=1e-12)
    assert np.all(np.abs(cs) <= 1 + 1e-15)
    assert np.allclose(_score(X * np.float32(4.0), q, COS), cs, rtol=1e-12)   # exact power-of-2 scaling
    assert np.allclose(_score(X, q * np.float32(2.0), IP), 2 * ip, rtol=0, atol=0)


def test_scores_vs_independent_numpy_fp64():
    """An independent numpy fp64 implementation (einsum, different reduction
    order) agrees to 1e-12 relative on small inputs, incl. odd d=1027 tail."""
    rng = np.random.default_rng(9)
    for d in (1, 8, 127, 1027):
        X = rng.standard_normal((20, d)).astype(np.float32)
        q = rng.standard_normal(d).astype(np.float32)
        X64, q64 = X.astype(np.float64), q.astype(np.float64)
        ip = np.einsum("ij,j->i", X64, q64)
        l2 = np.einsum("ij,ij->i", X64 - q64, X64 - q64)
        cs = ip / (np.linalg.norm(X64, axis=1) * np.linalg.norm(q64))
        for m, ref in ((IP, ip), (L2, l2), (COS, cs)):
            got = _score(X, q, m)
            assert np.allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


# -------------------------------------------------------------------- top-k

def _search(X, attrs, pred, Q, k, metric, off=0):
    X = np.asarray(X, dtype=np.float32)
    Q = np.atleast_2d(np.asarray(Q, dtype=np.float32))
    if attrs is None:
        attrs = [np.zeros(len(X), dtype=np.int32)]
    return oracle.search(X, attrs, pred, Q, k, metric, off)


@pytest.mark.parametrize("ex", GOLD["scan_per_tuple"], ids=lambda e: e["cite"][:24])
def test_spec_scan_examples(ex):
    if "cos" in ex:
        s = _score(ex["rows"], ex["query"], COS)
        assert np.allclose(s, ex["cos"], atol=1e-7)     # 0.8 is not exact in fp32
        return
    attrs = [np.array(ex["attr"], dtype=np.int32)] if "attr" in ex else None
    pred = [(0, ex["lo"], ex["hi"])] if "attr" in ex else []
    ids, dists, _ = _search(ex["rows"], attrs, pred, ex["query"], ex["k"], COS)
    assert ids[0].tolist() == ex["ids"]
    assert np.allclose(dists[0], ex["dists"], atol=1e-7)


@pytest.mark.parametrize("ex", GOLD["tensor_search"], ids=lambda e: e["cite"][:24])
def test_spec_tensor_examples(ex):
    attrs = [np.array(ex["attr"], dtype=np.int32)] if "attr" in ex else None
    pred = [(0, ex["lo"], ex["hi"])] if "attr" in ex else []
    ids, dists, _ = _search(ex["rows"], attrs, pred, ex["queries"], ex["k"], COS)
    assert ids.tolist() == ex["ids"]
    if "dists" in ex:
        assert np.allclose(dists, ex["dists"], atol=1e-7)
    else:
        assert np.all(np.isneginf(dists))               # COS padding is -inf


@pytest.mark.parametrize("ex", GOLD["extract_results"], ids=lambda e: e["cite"][:24])
def test_spec_extract_k_larger_than_m(ex):
    ids, dists, _ = _search(ex["rows"], None, [], ex["query"], ex["k"], COS)
    assert (ids[0] >= 0).sum() == ex["n_valid"]
    assert ids[0, ex["n_valid"]:].tolist() == [-1] * (ex["k"] - ex["n_valid"])


def test_order_orientation_and_padding_values():
    X = np.array([[0, 0], [1, 0], [3, 0], [2, 0]], dtype=np.float32)
    q = [0.5, 0]
    ids, d, _ = _search(X, None, [], q, 6, L2)
    assert ids[0].tolist() == [0, 1, 3, 2, -1, -1]            # ascending distance
    assert d[0].tolist()[:4] == [0.25, 0.25, 2.25, 6.25] and np.isposinf(d[0, 4:]).all()
    ids, d, _ = _search(X, None, [], q, 6, IP)
    assert ids[0].tolist() == [2, 3, 1, 0, -1, -1]            # descending inner product
    assert np.isneginf(d[0, 4:]).all()


def test_ties_go_to_lower_id():
    x = np.array([1, 2], dtype=np.float32)
    X = np.array([[5, 5], x, [9, 9], x, x], dtype=np.float32)    # rows 1,3,4 identical
    for m in (L2, IP, COS):
        ids, _, _ = _search(X, None, [], x if m == L2 else [1, 2], 5, m)
        pos = [ids[0].tolist().index(i) for i in (1, 3, 4)]
        assert pos == sorted(pos) and pos[1] == pos[0] + 1 and pos[2] == pos[1] + 1
    ids, d, _ = _search(X, None, [], x, 1, L2)
    assert ids[0].tolist() == [1] and d[0, 0] == 0.0         # identical vector distance 0


def test_exhaustive_permutations_tie_free():
    """Permuting the rows permutes the result ids and leaves the scores intact."""
    rng = np.random.default_rng(1)
    X = rng.standard_normal((6, 5)).astype(np.float32)
    q = rng.standard_normal(5).astype(np.float32)
    for m in (L2, IP, COS):
        ids0, d0, _ = _search(X, None, [], q, 4, m)
        for perm in itertools.permutations(range(6)):
            perm = np.array(perm)
            ids, d, _ = _search(X[perm], None, [], q, 4, m)
            assert perm[ids[0]].tolist() == ids0[0].tolist()
            assert d[0].tolist() == d0[0].tolist()


def test_brute_force_tiny_all_subsets():
    """For every subset of 7 rows (as a predicate on a row-index attribute)
    the result equals sorting the full result restricted to the subset."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((7, 3)).astype(np.float32)
    q = rng.standard_normal(3).astype(np.float32)
    attr = np.arange(7, dtype=np.int32)
    for m in (L2, IP):
        full, fd, _ = _search(X, [attr], [], q, 7, m)
        for lo in range(7):
            for hi in range(lo - 1, 7):
                ids, d, _ = _search(X, [attr], [(0, lo, hi)], q, 3, m)
                keep = [i for i in full[0].tolist() if lo <= i <= hi][:3]
                assert ids[0].tolist()[: len(keep)] == keep
                assert all(i == -1 for i in ids[0].tolist()[len(keep):])


def test_prefix_and_containment_and_selectivity_extremes():
    rng = np.random.default_rng(4)
    n, d = 500, 16
    X = rng.standard_normal((n, d)).astype(np.float32)
    a = rng.integers(0, 10, n).astype(np.int32)
    Q = rng.standard_normal((3, d)).astype(np.float32)
    for m in (L2, IP, COS):
        i10, _, _ = _search(X, [a], [(0, 0, 4)], Q, 10, m)
        i11, _, _ = _search(X, [a], [(0, 0, 4)], Q, 11, m)
        assert (i11[:, :10] == i10).all()                                   # prefix property
        iu, _, _ = _search(X, [a], [], Q, 10, m)
        for j in range(3):                                                  # containment
            qual = [i for i in iu[j] if 0 <= a[i] <= 4]
            assert set(qual) <= set(i10[j])
        iall, dall, _ = _search(X, [a], [(0, 0, 9)], Q, 10, m)              # s = 1 == unfiltered
        assert (iall == iu).all()
        inone, dnone, _ = _search(X, [a], [(0, 10, 20)], Q, 10, m)          # s = 0 -> padding
        assert (inone == -1).all()
        for j in range(3):                                                  # 100 % soundness
            assert all(0 <= a[i] <= 4 for i in i10[j])


def test_row_offset_and_shard_merge_decomposition():
    """top-k(union of shards) == merge(top-k per shard) -- north_star (4)."""
    rng = np.random.default_rng(6)
    n, d, k = 300, 8, 12
    X = rng.standard_normal((n, d)).astype(np.float32)
    a = rng.integers(0, 4, n).astype(np.int32)
    Q = rng.standard_normal((4, d)).astype(np.float32)
    cuts = [0, 97, 161, 300]
    for m in (L2, IP, COS):
        full_i, full_d, _ = _search(X, [a], [(0, 1, 2)], Q, k, m)
        parts_i, parts_d = [], []
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            i, dd, _ = _search(X[r0:r1], [a[r0:r1]], [(0, 1, 2)], Q, k, m, off=r0)
            assert ((i == -1) | ((i >= r0) & (i < r1))).all()
            parts_i.append(i)
            parts_d.append(dd)
        mi, md = oracle.merge(np.stack(parts_i), np.stack(parts_d), k, m)
        assert (mi == full_i).all() and (md == full_d).all()


def test_errors_mirror_abi():
    X = np.ones((3, 2), dtype=np.float32)
    a = np.zeros(3, dtype=np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.search(X, [a], [(1, 0, 0)], X[:1], 1, L2)
    assert e.value.status == oracle.ENOTFOUND
    with pytest.raises(oracle.OracleError) as e:
        oracle.search(X, [a], [], X[:1], 0, L2)
    assert e.value.status == oracle.EINVAL                          # k < 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.search(X, [a], [], X[:1], 1, 7)
    assert e.value.status == oracle.EINVAL                          # bad metric
    Z = X.copy()
    Z[1] = 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.search(Z, [a], [], X[:1], 1, COS)
    assert e.value.status == oracle.EDEGENERATE
    ids, d, _ = oracle.search(X, [a], [], np.zeros((1, 2), np.float32), 2, COS)
    assert (ids == -1).all()                                        # zero COS query -> padding
    ids, d, _ = oracle.search(X, [a], [], np.zeros((0, 2), np.float32), 2, L2)
    assert ids.shape == (0, 2)                                      # q = 0 no-op


def test_fp32_rounding_of_returned_dists():
    """dists are the fp64 scores rounded to nearest fp32."""
    rng = np.random.default_rng(8)
    X = rng.standard_normal((40, 33)).astype(np.float32)
    Q = rng.standard_normal((2, 33)).astype(np.float32)
    ids, d, s = _search(X, None, [], Q, 40, IP)
    assert (d == s.astype(np.float32)).all()
    assert np.all(np.diff(s, axis=1) <= 0)


# ---------------------------------------------------------------- range (threshold) selection
# orc_range: PAPER.md L354 ("cosine similarity > 0.9"), L1436 ("range instead of
# top-k"); SPEC.md L129-L133, L144 (ascending row id), L178 (>= tau); reading R14.

@pytest.mark.parametrize("ex", GOLD["range_search"], ids=lambda e: e["cite"][:24])
def test_spec_range_examples(ex):
    X = np.array(ex["rows"], dtype=np.float32)
    attrs = [np.array(ex.get("attr", [0] * len(X)), dtype=np.int32)]
    pred = [(0, ex["lo"], ex["hi"])] if "lo" in ex else []
    off, ids, dists, sc = oracle.range_search(X, attrs, pred, np.array([ex["query"]], dtype=np.float32), ex["tau"],
                                             COS)
    assert off.tolist() == [0, len(ex["ids"])]
    assert ids.tolist() == ex["ids"]
    assert np.allclose(dists, ex["dists"], atol=1e-7)


def _rand(n, d, seed, dup=False):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    if dup:
        X[n // 2] = X[0]
    attrs = [rng.integers(0, 10, n).astype(np.int32)]
    return rng, X, attrs


@pytest.mark.parametrize("metric", [L2, IP, COS])
def test_range_extremes_and_ascending_ids(metric):
    rng, X, attrs = _rand(300, 7, 11)
    Q = rng.standard_normal((3, 7)).astype(np.float32)
    pred = [(0, 2, 6)]
    _, _, sel = oracle.select(attrs, len(X), pred)
    everything = -np.inf if metric != L2 else np.inf
    nothing = np.inf if metric != L2 else -1.0
    off, ids, _, _ = oracle.range_search(X, attrs, pred, Q, everything, metric)
    assert off.tolist() == [0, len(sel), 2 * len(sel), 3 * len(sel)]
    for j in range(3):
        assert ids[off[j]:off[j + 1]].tolist() == sel.tolist()      # every qualifying row, ascending
    off, ids, _, _ = oracle.range_search(X, attrs, pred, Q, nothing, metric)
    assert off.tolist() == [0, 0, 0, 0] and len(ids) == 0


@pytest.mark.parametrize("metric", [L2, IP, COS])
def test_range_equals_independent_numpy_filter(metric):
    """Brute force with numpy fp64 (independent of the C oracle's loops)."""
    rng, X, attrs = _rand(257, 13, 12)
    Q = rng.standard_normal((4, 13)).astype(np.float32)
    pred = [(0, 0, 4)]
    keep_row = (attrs[0] >= 0) & (attrs[0] <= 4)
    Xd, Qd = X.astype(np.float64), Q.astype(np.float64)
    if metric == L2:
        S = ((Qd[:, None, :] - Xd[None, :, :]) ** 2).sum(-1)
    elif metric == IP:
        S = Qd @ Xd.T
    else:
        S = (Qd @ Xd.T) / np.linalg.norm(Qd, axis=1)[:, None] / np.linalg.norm(Xd, axis=1)[None, :]
    tau = float(np.median(S))
    off, ids, _, sc = oracle.range_search(X, attrs, pred, Q, tau, metric)
    for j in range(4):
        want = np.nonzero(keep_row & ((S[j] <= tau) if metric == L2 else (S[j] >= tau)))[0]
        assert ids[off[j]:off[j + 1]].tolist() == want.tolist()
        assert np.allclose(sc[off[j]:off[j + 1]], S[j, want], rtol=1e-12)


@pytest.mark.parametrize("metric", [L2, IP, COS])
def test_range_containment_and_monotone_in_tau(metric):
    rng, X, attrs = _rand(400, 9, 13)
    Q = rng.standard_normal((2, 9)).astype(np.float32)
    _, _, sc = oracle.search(X, attrs, [], Q, 50, metric)
    lo_tau, hi_tau = float(np.median(sc[:, 20])), float(np.median(sc[:, 40]))   # two thresholds
    a = oracle.range_search(X, attrs, [(0, 3, 8)], Q, lo_tau, metric)
    b = oracle.range_search(X, attrs, [], Q, lo_tau, metric)
    c = oracle.range_search(X, attrs, [], Q, hi_tau, metric)
    _, _, sel = oracle.select(attrs, len(X), [(0, 3, 8)])
    for j in range(2):
        fa, fb, fc = (set(r[1][r[0][j]:r[0][j + 1]].tolist()) for r in (a, b, c))
        assert fa == fb & set(sel.tolist())          # result(theta) = result(no theta) n sigma_theta
        strict, loose = (fb, fc) if (metric == L2) == (lo_tau < hi_tau) else (fc, fb)
        assert strict <= loose                       # monotone in tau


@pytest.mark.parametrize("metric", [L2, IP, COS])
def test_range_at_kth_score_equals_topk(metric):
    """Tie-free data: the range result at tau = the k-th best score is the top-k set."""
    rng, X, attrs = _rand(500, 16, 14)
    Q = rng.standard_normal((3, 16)).astype(np.float32)
    k = 17
    tk_ids, _, tk_sc = oracle.search(X, attrs, [(0, 1, 9)], Q, k, metric)
    for j in range(3):
        off, ids, _, _ = oracle.range_search(X, attrs, [(0, 1, 9)], Q[j:j + 1], float(tk_sc[j, k - 1]), metric)
        assert sorted(ids.tolist()) == sorted(tk_ids[j].tolist()) and len(ids) == k


def test_range_l2_duplicate_row_at_zero_and_cos_zero_query():
    rng, X, attrs = _rand(64, 5, 15, dup=True)
    off, ids, dists, _ = oracle.range_search(X, attrs, [], X[:1], 0.0, L2)
    assert ids.tolist() == [0, 32] and dists.tolist() == [0.0, 0.0]
    Qz = np.zeros((1, 5), dtype=np.float32)
    off, ids, _, _ = oracle.range_search(X, attrs, [], Qz, -1.0, COS)
    assert off.tolist() == [0, 0]
