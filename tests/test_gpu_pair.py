"""The main pass as CTA pairs (tc_kernel.cuh PAIR: a cluster of two CTAs -- query tiles
2i, 2i + 1 of a row split -- each staging half of every row tile, one cta_group::2
M = 256 MMA per K step): parity with the oracle for every row delivery (masked tiles,
the X_sel copy by TMA, cp.async by id), every metric, ragged query / row tails and an
odd tile count (no pairing).  Environment switches are read once per process, so each
variant runs in a subprocess (with a time limit: a pairing bug shows as a hang)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle, paper_2403_15807_b200 as vrs
from parity import check_topk
M = {oracle.L2: "l2", oracle.IP: "ip", oracle.COS: "cos"}
cases = [(20000, 256, 256, 10, oracle.IP, [(0, 0, 99)]),       # 2 query tiles, 10 %
         (30011, 768, 200, 100, oracle.L2, [(0, 0, 499)]),     # ragged second tile, 50 %
         (9000, 1536, 512, 50, oracle.COS, [(0, 0, 899)]),     # 4 tiles = 2 pairs, 90 %
         (12000, 256, 300, 10, oracle.IP, [(0, 0, 299)]),      # 3 tiles: no pairing
         (5000, 512, 129, 20, oracle.L2, [(0, 5000, 6000)]),   # empty selection
         (777, 256, 160, 240, oracle.IP, [(0, 0, 999)])]       # one partial row tile, k > N_sel / 4
for n, d, q, k, metric, pred in cases:
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
    for rows in (None, 1, 2):
        ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=M[metric], path=vrs.PATH_GEMM, rows=rows)
        torch.cuda.synchronize()
        check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric)
    del ix
print("OK")
'''


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]


def test_pair_default_delivery():
    _run({"VRS_PAIR": "1"})


def test_pair_cp_async():
    """cp.async by id for <= 2 query tiles at any selection size (VRS_CP_MIN_MB=0)."""
    _run({"VRS_PAIR": "1", "VRS_CP_MIN_MB": "0"})


def test_pair_off():
    _run({"VRS_PAIR": "0"})
