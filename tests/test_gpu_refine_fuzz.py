"""The refine pass forced on every fp16 tensor-core search
(VRS_REFINE=always, VRS_REFINE_QMIN=1; read once per process, so a subprocess):
seeded random shapes, metrics, k, row delivery (auto / masked / gathered, with the
X_sel copy, cp.async by id, and the refine's X_sel_lo), clustered data (many
uncertified queries: the fold over few active tiles) and Gaussian data (none: the
refine runs with a zero count and must change nothing).  Results must be the
oracle's exactly (check_topk_exact), whatever fraction the refine certifies."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle, paper_2403_15807_b200 as vrs
from parity import check_topk_exact
M = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}
refined = 0
for seed in range(int(sys.argv[2])):
    rng = np.random.default_rng(int(os.environ.get('VRS_FUZZ_BASE', '0')) + 4000 + seed)   # (soak runs: fresh seeds)
    n = int(rng.integers(2000, 60000))
    d = int(rng.choice([8, 64, 72, 128, 256, 320]))
    q = int(rng.choice([1, 5, 64, 128, 130, 300, 700]))
    k = int(rng.choice([1, 10, 30, 50]))
    metric = int(rng.choice([oracle.L2, oracle.IP, oracle.COS]))
    clustered = bool(rng.integers(0, 4))
    if clustered:
        C = int(rng.integers(4, 40))
        cent = rng.standard_normal((C, d)).astype(np.float32)
        cid = rng.integers(0, C, n)
        X = (cent[cid] + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
        Q = (cent[rng.integers(0, C, q)] + 0.05 * rng.standard_normal((q, d))).astype(np.float32)
    else:
        X = rng.standard_normal((n, d)).astype(np.float32)
        Q = rng.standard_normal((q, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    lo = int(rng.integers(0, 900))
    pred = [] if rng.integers(0, 3) == 0 else [(0, lo, int(rng.integers(lo, 1000)))]
    rows = [None, vrs.ROWS_MASKED, vrs.ROWS_GATHER][int(rng.integers(0, 3))]
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs],
                   precision=vrs.PREC_FP16)
    st = vrs.new_stats()
    ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=M[metric], path=vrs.PATH_GEMM, rows=rows,
                           stats=st)
    torch.cuda.synchronize()
    s = vrs.read_stats(st)
    try:
        check_topk_exact(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric)
    except AssertionError as e:
        raise AssertionError(f"seed {seed}: n={n} d={d} q={q} k={k} metric={metric} clustered={clustered} "
                             f"pred={pred} rows={rows} stats={s}: {e}")
    assert s["max_key_error_over_bound"] < 1.0, (seed, s)
    refined += s["refined"]
    del ix
print("REFINED", refined)
print("OK")
'''


def test_refine_forced_fuzz(vrs_lib_built):
    env = dict(os.environ, VRS_REFINE="always", VRS_REFINE_QMIN="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, "100"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]
    # the clustered cases must have exercised the refine itself, not only its zero-count launch
    refined = int(r.stdout.split("REFINED")[1].split()[0])
    assert refined > 0, r.stdout[-2000:]


@pytest.fixture(scope="module")
def vrs_lib_built():
    import paper_2403_15807_b200 as m
    m.library()
    return m
