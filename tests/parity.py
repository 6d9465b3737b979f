"""GPU-vs-oracle acceptance rules (from BASELINE.json north_star):
bitmap / count bit-exact; exactly min(k, N_sel) valid entries with exact padding;
ids unique, in range, 100 % qualifying; every returned dist within 1e-3 relative of
the oracle's fp64 score of that id and of the oracle's dist at the same rank; id sets
identical except rows whose oracle score lies within 1e-3 relative of the k-th.
On top of these (check_topk exact=True, the default), the certified-exact contract
of DESIGN.md Sec. 7: ids identical to the oracle's rank for rank and dists equal to
fp32(oracle fp64) within one ulp (check_topk_exact)."""
import numpy as np

import oracle

RTOL = 1e-3          # north_star: "Distances must agree within 1e-3 relative error"


def check_select(bitmap_dev, count_dev, ids_dev, attrs_np, n, pred):
    rb, rc, rids = oracle.select(attrs_np, n, pred)
    gb = bitmap_dev.cpu().numpy().view(np.uint32)
    assert gb.shape == rb.shape and (gb == rb).all(), "bitmap words differ"
    assert int(count_dev.cpu()[0]) == rc, f"count {int(count_dev.cpu()[0])} != {rc}"
    if ids_dev is not None:
        assert (ids_dev.cpu().numpy()[:rc] == rids).all(), "compacted ids differ"
    return rc


def check_topk(gi, gd, X, attrs_np, pred, Q, k, metric, row_offset=0, ref=None, rtol=RTOL, exact=True):
    """gi, gd: numpy [q, k] from the GPU.  X, Q: numpy fp32.  Returns #queries checked."""
    if ref is None:
        ref = oracle.search(X, attrs_np, pred, Q, k, metric, row_offset)
    rid, rd, rs = ref
    n = X.shape[0]
    _, cnt, qual = oracle.select(attrs_np, n, pred)
    qual_set = set((qual + row_offset).tolist())
    pad = np.inf if metric == oracle.L2 else -np.inf
    for j in range(Q.shape[0]):
        m = int((rid[j] >= 0).sum())
        assert int((gi[j] >= 0).sum()) == m, f"q{j}: {int((gi[j] >= 0).sum())} valid entries, oracle {m}"
        assert (gi[j, m:] == -1).all() and (gd[j, m:] == pad).all(), f"q{j}: bad padding"
        if m == 0:
            continue
        v = gi[j, :m]
        assert len(set(v.tolist())) == m, f"q{j}: duplicate ids"
        assert set(v.tolist()) <= qual_set, f"q{j}: returned a row that fails the predicate"
        s = oracle.score(X, Q[j], v - row_offset, metric)
        err = np.abs(gd[j, :m].astype(np.float64) - s)
        assert (err <= rtol * np.abs(s)).all(), f"q{j}: dist vs own oracle score, max rel {np.max(err / np.abs(s))}"
        err2 = np.abs(gd[j, :m].astype(np.float64) - rs[j, :m])
        assert (err2 <= rtol * np.abs(rs[j, :m])).all(), f"q{j}: dist vs oracle at same rank"
        sk = rs[j, m - 1]
        diff = set(v.tolist()) ^ set(rid[j, :m].tolist())
        if diff:
            ds = oracle.score(X, Q[j], np.array(sorted(diff)) - row_offset, metric)
            assert (np.abs(ds - sk) <= rtol * abs(sk)).all(), f"q{j}: id sets differ outside the k-th band"
    if exact:   # the certified-exact contract on top of north_star's band rules
        check_topk_exact(gi, gd, X, attrs_np, pred, Q, k, metric, row_offset, ref=ref)
    return Q.shape[0]


def check_topk_exact(gi, gd, X, attrs_np, pred, Q, k, metric, row_offset=0, ref=None, tie_rtol=1e-12):
    """Certified exactness: the GPU result IS the oracle's result.
    Every rank holds the oracle's id -- two rows may trade places only when their fp64
    oracle scores agree to tie_rtol (the GPU sums in another order) -- and every dist
    is fp32(the oracle's fp64 score) within one ulp (the rounding boundary can fall
    between the two fp64 sums).  Padding as in check_topk."""
    if ref is None:
        ref = oracle.search(X, attrs_np, pred, Q, k, metric, row_offset)
    rid, rd, rs = ref
    pad = np.inf if metric == oracle.L2 else -np.inf
    bad = []
    for j in range(Q.shape[0]):
        m = int((rid[j] >= 0).sum())
        assert int((gi[j] >= 0).sum()) == m, f"q{j}: {int((gi[j] >= 0).sum())} valid entries, oracle {m}"
        assert (gi[j, m:] == -1).all() and (gd[j, m:] == pad).all(), f"q{j}: bad padding"
        if m == 0:
            continue
        g = gi[j, :m]
        assert len(set(g.tolist())) == m, f"q{j}: duplicate ids"
        sg = oracle.score(X, Q[j], g - row_offset, metric)
        scale = np.maximum(np.abs(rs[j, :m]), 1e-300)
        moved = g != rid[j, :m]
        if moved.any() and not (np.abs(sg[moved] - rs[j, :m][moved]) <= tie_rtol * scale[moved]).all():
            bad.append((j, int(np.argmax(moved)), g[moved][:4].tolist(), rid[j, :m][moved][:4].tolist()))
            continue
        ulp = np.spacing(np.abs(rd[j, :m]).astype(np.float32))
        err = np.abs(gd[j, :m].astype(np.float64) - rd[j, :m].astype(np.float64))
        assert (err <= ulp).all(), f"q{j}: dist more than 1 ulp from fp32(oracle fp64), max {np.max(err / ulp)} ulp"
    assert not bad, f"{len(bad)} queries differ from the oracle's ids, e.g. (query, rank, gpu, oracle) {bad[:3]}"
    return Q.shape[0]
