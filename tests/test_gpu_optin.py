"""The opt-in variants of the tensor-core path (environment switches read once per
process, so each runs in a subprocess): TMA gather4 late materialisation
(VRS_GATHER4), cp.async gathering straight into the swizzled stages
(VRS_CPGATHER), the one-launch selection + select_finish (VRS_SELECT_LOCAL), the
small-batch finalize variants (VRS_FIN_STAGE, VRS_FIN_BLOCK_Q) and the
warp-voted slow path (libvrs_exp.so, -DVRS_SLOW_GROUPS_VOTE, when built).  Each
must meet the same parity rules as the default path."""
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
cases = [(20000, 128, 300, 10, oracle.IP, [(0, 0, 99)]),       # gathered, 10 %
         (12000, 64, 700, 50, oracle.COS, [(0, 0, 299)]),      # gathered, q >= 592
         (9000, 768, 9, 100, oracle.L2, [(0, 0, 299)]),        # d = 768, 30 %
         (6000, 128, 64, 10, oracle.L2, [(0, 5000, 6000)]),    # empty selection
         (200000, 128, 16, 10, oracle.IP, [(0, 0, 899)])]      # 90 %, >= 2 x 148 row tiles: cp.async (cp_fetch)
for n, d, q, k, metric, pred in cases:
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 1000, n).astype(np.int32)]
    Q = rng.standard_normal((q, d)).astype(np.float32)
    for rows, prec in ((None, None), (2, None), (2, 1)):
        ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs], precision=prec)
        ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric=M[metric], path=vrs.PATH_GEMM, rows=rows)
        torch.cuda.synchronize()
        check_topk(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, metric)
        del ix
    # range mode through the same selection / row delivery
    if metric != oracle.L2:
        ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
        off, rid, rd = ix.range_search(torch.from_numpy(Q[:4]).cuda(), pred, tau=0.5 if metric == oracle.COS else 8.0,
                                       metric=M[metric])
        o_off, o_ids, o_d, _ = oracle.range_search(X, attrs, pred, Q[:4], 0.5 if metric == oracle.COS else 8.0, metric)
        assert np.array_equal(off.cpu().numpy(), o_off) and np.array_equal(rid.cpu().numpy(), o_ids)
print("OK")
'''


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]


def test_gather4(vrs_lib_built):
    _run({"VRS_GATHER4": "1"})


def test_cp_async_gather(vrs_lib_built):
    _run({"VRS_CPGATHER": "1"})


def test_cp_gather_adaptive_threshold(vrs_lib_built):
    """The default device-side choice between the X_sel copy and cp.async (one query
    tile, selection >= the threshold), with the threshold lowered to 1 MB so that the
    cases above take both branches (the gather copy kernel skips itself by the same test)."""
    _run({"VRS_CP_MIN_MB": "1"})


def test_select_local(vrs_lib_built):
    _run({"VRS_SELECT_LOCAL": "1"})


def test_finalize_block_radix(vrs_lib_built):
    """The small-batch block finalize with its histogram selection skipped: the radix
    select over the staged candidates (the path for one-valued keys / crowded buckets)."""
    _run({"VRS_FIN_STAGE": "-1"})


def test_finalize_block_unstaged(vrs_lib_built):
    """The small-batch block finalize with staging capped at one candidate: the radix
    select reads the lists in global memory (the path for > kFinStage candidates)."""
    _run({"VRS_FIN_STAGE": "1"})


def test_finalize_cta_small_q(vrs_lib_built):
    """Small batches through the 8/16-warp CTA finalize instead of the block finalize."""
    _run({"VRS_FIN_BLOCK_Q": "0"})


def test_slow_path_vote_variant(vrs_lib_built):
    if not os.path.exists(os.path.join(ROOT, "paper_2403_15807_b200", "libvrs_exp.so")):
        pytest.skip("libvrs_exp.so not built (make exp)")
    _run({"VRS_LIB": "exp"})


@pytest.fixture(scope="module")
def vrs_lib_built():
    import paper_2403_15807_b200 as m
    m.library()
    return True
