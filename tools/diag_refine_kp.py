"""Refine-pass certification vs k' (diagnostic): clustered cosine data (C5-like), the
level-0 / refine / exact-fallback counts from the stats block, parity vs the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2403_15807_b200 as vrs  # noqa: E402
from parity import check_topk_exact  # noqa: E402

rng = np.random.default_rng(5)
n, d, C = 200_000, 256, 64
cent = rng.standard_normal((C, d)).astype(np.float32)
cid = rng.integers(0, C, n)
X = (cent[cid] + 0.1 * rng.standard_normal((n, d))).astype(np.float32)
attrs = [(cid + rng.integers(0, 8, n)).astype(np.int32)]
Q = (cent[rng.integers(0, C, 256)] + 0.1 * rng.standard_normal((256, d))).astype(np.float32)
ix = vrs.Index(torch.from_numpy(X).cuda(), [torch.from_numpy(a).cuda() for a in attrs])
for k in [int(x) for x in sys.argv[1:]] or [50]:
    for pred in ([(0, 7, 30)], [(0, 7, 7)]):
        st = vrs.new_stats()
        ids, dists = ix.search(torch.from_numpy(Q).cuda(), pred, k=k, metric="cos", stats=st)
        torch.cuda.synchronize()
        s = vrs.read_stats(st)
        check_topk_exact(ids.cpu().numpy(), dists.cpu().numpy(), X, attrs, pred, Q, k, oracle.COS)
        print(f"k={k} pred={pred} kprime_env={os.environ.get('VRS_KPRIME')} stats={s} parity ok")
