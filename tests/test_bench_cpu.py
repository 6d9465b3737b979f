"""bench.py host logic without a GPU: the workload descriptions, the torchrun relaunch
command for --gpus N, and the oracle-merge parity reduction used at N > 1."""
import os
import sys

import numpy as np

import datagen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_default_workload_is_c4_weak_scaling():
    old = sys.argv
    sys.argv = ["bench.py"]
    try:
        args = bench.parse()
    finally:
        sys.argv = old
    assert args.workload == "c4" and args.gpus == 1 and args.warmup >= 3
    cfg = datagen.CONFIGS[args.workload]
    for world in (1, 2, 4, 8):
        d = bench.workload_desc(cfg, world)
        assert d["n"] == 6_250_000 * world and d["rows_per_gpu"] == 6_250_000
    assert bench.workload_desc(cfg, 1)["queries_per_step"] == 3 * (1 + 256 + 8192)


def test_relaunch_command(monkeypatch):
    """--gpus N outside torchrun re-executes under torch.distributed.run with N ranks on 127.0.0.1."""
    seen = {}

    def fake_execv(exe, cmd):
        seen["exe"], seen["cmd"] = exe, cmd
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    args = bench.parse()
    try:
        bench.relaunch_distributed(args)
    except SystemExit:
        pass
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_multi_gpu_parity_reduction():
    """At N > 1 every rank computes its shard's oracle top-k and rank 0 merges them with the
    oracle's merge: equal to the oracle on the whole corpus (the decomposition bench relies on)."""
    rng = np.random.default_rng(3)
    n, d, k = 3000, 16, 7
    X = rng.standard_normal((n, d)).astype(np.float32)
    attrs = [rng.integers(0, 100, n).astype(np.int32)]
    Q = rng.standard_normal((4, d)).astype(np.float32)
    pred = [(0, 0, 49)]
    for metric in (oracle.L2, oracle.IP, oracle.COS):
        ri, rd, _ = oracle.search(X, attrs, pred, Q, k, metric)
        cuts = [0, 1000, 2000, 3000]
        parts_i, parts_d = [], []
        for a, b in zip(cuts[:-1], cuts[1:]):
            pi, pd, _ = oracle.search(X[a:b], [c[a:b] for c in attrs], pred, Q, k, metric, row_offset=a)
            parts_i.append(pi)
            parts_d.append(pd)
        mi, md = oracle.merge(np.stack(parts_i), np.stack(parts_d), k, metric)
        assert (mi == ri).all() and (md == rd).all()
        gi, gd = bench.compare_exact(mi, md, ri, rd)
        assert gi == 0 and gd == 0
