"""Row-sharded multi-GPU search (north_star (4)).

One process per GPU (torchrun), NCCL process group.  Rank r owns the
contiguous rows [r*N/G, (r+1)*N/G) of the corpus (global id = row_offset +
local id); the queries and the predicate are replicated.  Each rank runs the
whole single-GPU path on its shard (vrs_search -> exact [Q x k] dists and
global ids); one all-gather of each output array over NCCL (NVLink 5 /
NVSwitch) and vrs_merge on every rank give the identical global top-k
(top-k is decomposable under the (dist, id) total order).  PeerMerge does the exchange
and the merge in one kernel over peer (symmetric) memory instead (vrs_merge_push).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int):
    """Contiguous row range [r0, r1) of `rank` (sizes differ by at most one row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    return n * rank // world, n * (rank + 1) // world


def all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """[q, k] on every rank -> [world, q, k] (rank-major), same on every rank."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    try:
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    except (RuntimeError, NotImplementedError, AttributeError):
        parts = list(out.unbind(0))
        dist.all_gather(parts, t.contiguous(), group=group)
    return out


def gather_merge(ids: torch.Tensor, dists: torch.Tensor, k: int, metric, group=None, merge_fn=None):
    """All-gather every rank's exact local top-k and merge (vrs_merge by default)."""
    if merge_fn is None:
        from . import merge as merge_fn
    gi = all_gather_rows(ids, group)
    gd = all_gather_rows(dists, group)
    return merge_fn(gi, gd, k, metric)


class PeerMerge:
    """The exchange + merge as one kernel over peer memory (vrs_merge_push): every rank
    allocates a receive buffer of vrs_push_buffer_bytes(world, q_max, k) in torch symmetric
    memory (peer-mapped over NVLink), rendezvous once, then each merge() pushes the rank's
    [q x k] results into every rank's buffer and merges its own -- one launch per call, no
    NCCL collective, CUDA-graph capturable.  Raises if symmetric memory is unavailable
    (callers fall back to gather_merge)."""

    def __init__(self, q_max: int, k: int, group=None, device=None):
        import ctypes

        import torch.distributed._symmetric_memory as symm_mem

        from . import library
        self.lib = library()
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.k, self.q_max = int(k), int(q_max)
        self.bytes = int(self.lib.vrs_push_buffer_bytes(self.world, self.q_max, self.k))
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.buf = symm_mem.empty((self.bytes + 7) // 8, dtype=torch.int64, device=dev)
        self.buf.zero_()   # (the per-source push counts start at 0)
        torch.cuda.synchronize(dev)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        self.peer_ptrs = ctypes.c_void_p(int(self.handle.buffer_ptrs_dev))
        self.state = torch.zeros(4, dtype=torch.int32, device=dev)
        dist.barrier(group=self.group)

    def merge(self, ids: torch.Tensor, dists: torch.Tensor, metric, out=None, stream=None):
        from . import _lib, _metric, _ptr, _stream
        q, k = ids.shape
        if k != self.k or q > self.q_max:
            raise ValueError(f"PeerMerge sized for q <= {self.q_max}, k = {self.k}")
        oi, od = out if out is not None else (torch.empty_like(ids), torch.empty_like(dists))
        st = self.lib.vrs_merge_push(_ptr(ids.contiguous()), _ptr(dists.contiguous()), self.peer_ptrs, self.bytes,
                                     self.world, self.rank, q, k, _metric(metric), _ptr(self.state), _ptr(oi),
                                     _ptr(od), _stream(stream))
        _lib.check(st, "vrs_merge_push")
        return oi, od

    def timed_out(self) -> bool:
        """True once a call's wait for a peer's push expired (vrs.h: state[3]); synchronises.
        Every output since is invalid -- the caller falls back to gather_merge."""
        return bool(self.state[3].item() != 0)

    def validate(self, metric="ip") -> bool:
        """One exchange of a deterministic [q_max x k] pattern through the push kernel AND
        through gather_merge (NCCL all-gather + vrs_merge); True iff every rank got identical
        results and no wait expired.  Collective: every rank calls it.  Run once before trusting
        the peer transport (e.g. a first multi-GPU box)."""
        dev = self.state.device
        q, k = self.q_max, self.k
        g = torch.Generator(device="cpu").manual_seed(1234 + self.rank)
        from . import _metric
        best_first_desc = int(_metric(metric)) != 0   # (VRS_L2 = 0: smaller is better)
        d = torch.randn(q, k, generator=g).sort(dim=1, descending=best_first_desc).values.to(dev)
        i = (torch.arange(q * k, dtype=torch.int64).reshape(q, k) * self.world + self.rank).to(dev)
        gi, gd = self.merge(i, d, metric)
        ri, rd = gather_merge(i, d, k, metric, self.group)
        ok = torch.equal(gi, ri) and torch.equal(gd, rd) and not self.timed_out()
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return bool(flag.item())


class ShardedIndex:
    """The calling rank's shard of a row-sharded corpus."""

    def __init__(self, vectors: torch.Tensor, attrs, row_offset: int, group=None):
        from . import Index
        self.group = group
        self.local = Index(vectors, attrs, row_offset=row_offset)

    def search(self, queries, pred=None, k: int = 10, metric="l2", path=None, rows=None):
        ids, dists = self.local.search(queries, pred, k=k, metric=metric, path=path, rows=rows)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            return gather_merge(ids, dists, k, metric, self.group)
        return ids, dists
