"""vrs_merge_push (the exchange + merge in one kernel over torch symmetric memory) on the
one GPU a test box has: a world-size-1 NCCL group, so the push goes to the rank's own
buffer -- the kernel's slot layout, push counts, epoch / parity bookkeeping across calls
and across CUDA-graph replays, and its merge (vs vrs_merge) are exercised; the NVLink
transport itself needs a multi-GPU box."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, socket, sys, numpy as np, torch
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_2403_15807_b200 as vrs
from paper_2403_15807_b200.dist import PeerMerge
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
rng = np.random.default_rng(3)
q_max, k = 300, 20
pm = PeerMerge(q_max, k)

def case(q, metric):
    d = rng.standard_normal((q, k)).astype(np.float32)
    i = rng.permutation(10 ** 6)[: q * k].reshape(q, k).astype(np.int64)
    i[:, -3:] = -1                                   # padding entries
    d[:, -3:] = np.inf if metric == "l2" else -np.inf
    return torch.from_numpy(i).cuda(), torch.from_numpy(d).cuda()

for metric in ("l2", "ip", "cos"):
    for q in (1, 7, 300, 150):                       # several calls: epochs 1.., both parities
        ids, dists = case(q, metric)
        gi, gd = pm.merge(ids, dists, metric)
        ri, rd = vrs.merge(ids[None], dists[None], k, metric)
        torch.cuda.synchronize()
        assert torch.equal(gi, ri) and torch.equal(gd, rd), (metric, q)
# CUDA graph: the epoch lives in device memory, so replays advance it
ids, dists = case(64, "ip")
out = (torch.empty(64, k, dtype=torch.int64, device="cuda"), torch.empty(64, k, device="cuda"))
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    pm.merge(ids, dists, "ip", out=out)
torch.cuda.current_stream().wait_stream(st)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    pm.merge(ids, dists, "ip", out=out)
for rep in range(5):
    ni, nd = case(64, "ip")
    ids.copy_(ni); dists.copy_(nd)
    g.replay()
    ri, rd = vrs.merge(ids[None], dists[None], k, "ip")
    torch.cuda.synchronize()
    assert torch.equal(out[0], ri) and torch.equal(out[1], rd), rep
assert not pm.timed_out()
assert pm.validate("ip") and pm.validate("l2")     # push kernel == all-gather + vrs_merge, no expired wait
dist.destroy_process_group()
print("OK")
'''


def test_peer_merge_world1():
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]


TIMEOUT_SCRIPT = r'''
import ctypes, sys, time, torch
sys.path.insert(0, sys.argv[1])
import paper_2403_15807_b200 as vrs
lib = vrs.library()
torch.cuda.set_device(0)
q, k, parts = 40, 10, 2
nbytes = int(lib.vrs_push_buffer_bytes(parts, q, k))
bufs = [torch.zeros((nbytes + 7) // 8, dtype=torch.int64, device="cuda") for _ in range(parts)]
ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
state = torch.zeros(4, dtype=torch.int32, device="cuda")
ids = torch.arange(q * k, dtype=torch.int64, device="cuda").reshape(q, k)
dists = torch.randn(q, k, device="cuda").sort(dim=1, descending=True).values
oi, od = torch.empty_like(ids), torch.empty_like(dists)
P = lambda t: ctypes.c_void_p(t.data_ptr())
torch.cuda.synchronize()
t0 = time.time()
st = lib.vrs_merge_push(P(ids), P(dists), P(ptrs), nbytes, parts, 0, q, k, 1, P(state), P(oi), P(od),
                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
assert st == 0, st
torch.cuda.synchronize()
dt = time.time() - t0
# rank 1 never pushes: the wait for its pushes expires (VRS_PUSH_TIMEOUT_MS = 300) and the flag is set
assert state[3].item() == 1, state.tolist()
assert 0.25 < dt < 10.0, dt
print("OK")
'''


def test_push_wait_is_bounded():
    """A peer that never pushes: the kernel gives up after the wait bound and sets state[3]
    (vrs.h) instead of hanging the GPU.  (One rank, two plain device buffers: no peer kernel
    is waited for -- the point is that none arrives.)"""
    env = dict(os.environ, VRS_PUSH_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", TIMEOUT_SCRIPT, ROOT], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-4000:]
