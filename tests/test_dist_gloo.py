"""World-size-2 gloo test of the row-sharded search's host logic on CPU:
shard ranges, global ids via row_offset, the all-gather layout and the merge
give exactly the single-process global top-k.  Per-shard search and the merge
are supplied by the oracle here (no GPU); on the GPU box the same
paper_2403_15807_b200.dist.gather_merge runs with vrs_search / vrs_merge."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_merge(gi, gd, k, metric):
    i, d = oracle.merge(gi.numpy(), gd.numpy(), k, metric)
    return torch.from_numpy(i), torch.from_numpy(d)


def _worker(rank, port, out_dir, name, n, sel):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2403_15807_b200.dist import gather_merge, shard_range
    cfg = datagen.CONFIGS[name]
    r0, r1 = shard_range(n, WORLD, rank)
    X, attrs = datagen.corpus(cfg, r0, r1, "cpu", n=n, d=32)
    Q = datagen.queries(cfg, 5, "cpu", d=32)
    pred = datagen.predicate(cfg, sel)
    ids, dists, _ = oracle.search(X.numpy(), [a.numpy() for a in attrs], pred, Q.numpy(), cfg.k, cfg.metric,
                                  row_offset=r0)
    mi, md = gather_merge(torch.from_numpy(ids), torch.from_numpy(dists), cfg.k, cfg.metric,
                          merge_fn=_oracle_merge)
    np.save(os.path.join(out_dir, f"ids{rank}.npy"), mi.numpy())
    np.save(os.path.join(out_dir, f"d{rank}.npy"), md.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n,sel", [("c2", 20_001, 0.1), ("c5", 12_345, 0.01), ("c1", 10_000, 0.1)])
def test_sharded_merge_equals_global(name, n, sel):
    cfg = datagen.CONFIGS[name]
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_worker, args=(_free_port(), tmp, name, n, sel), nprocs=WORLD, start_method="spawn")
        X, attrs = datagen.corpus(cfg, 0, n, "cpu", n=n, d=32)
        Q = datagen.queries(cfg, 5, "cpu", d=32)
        ref_i, ref_d, _ = oracle.search(X.numpy(), [a.numpy() for a in attrs], datagen.predicate(cfg, sel),
                                        Q.numpy(), cfg.k, cfg.metric)
        for r in range(WORLD):
            assert (np.load(os.path.join(tmp, f"ids{r}.npy")) == ref_i).all()
            assert (np.load(os.path.join(tmp, f"d{r}.npy")) == ref_d).all()


def test_shard_ranges_cover_exactly():
    from paper_2403_15807_b200.dist import shard_range
    for n in (1, 7, 50_000_000, 10_000_000, 1_000_000):
        for world in (1, 2, 4, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(r1 - r0 for r0, r1 in rs) - min(r1 - r0 for r0, r1 in rs) <= 1


def _fallback_worker(rank, port, out_dir):
    """The bench's exchange at N > 1 without symmetric memory (here: gloo on CPU):
    PeerMerge refuses, gather_merge carries the exchange."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2403_15807_b200.dist import PeerMerge, gather_merge
    ok = False
    try:
        PeerMerge(16, 10)
    except Exception:   # noqa: BLE001 -- expected without CUDA symmetric memory
        ok = True
    rng = np.random.default_rng(rank)
    d = np.sort(rng.standard_normal((4, 10)).astype(np.float32), axis=1)
    i = (rank * 1000 + np.arange(40)).reshape(4, 10).astype(np.int64)
    mi, md = gather_merge(torch.from_numpy(i), torch.from_numpy(d), 10, oracle.L2, merge_fn=_oracle_merge)
    np.save(os.path.join(out_dir, f"fb{rank}.npy"), np.array([ok]))
    np.save(os.path.join(out_dir, f"fi{rank}.npy"), mi.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_peer_merge_falls_back_without_symmetric_memory():
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_fallback_worker, args=(_free_port(), tmp), nprocs=WORLD, start_method="spawn")
        for r in range(WORLD):
            assert np.load(os.path.join(tmp, f"fb{r}.npy"))[0]
        assert np.array_equal(np.load(os.path.join(tmp, "fi0.npy")), np.load(os.path.join(tmp, "fi1.npy")))


def test_push_buffer_layout():
    """vrs_push_buffer_bytes: a 256-byte count header + 2 parities x parts x q x k x (8 + 4) bytes."""
    import paper_2403_15807_b200 as vrs
    lib = vrs.library()
    for parts, q, k in ((1, 1, 1), (8, 25347, 100), (2, 4096, 10)):
        assert lib.vrs_push_buffer_bytes(parts, q, k) == 256 + 2 * parts * q * k * 12
