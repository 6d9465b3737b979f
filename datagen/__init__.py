"""Seeded synthetic inputs shared by the product tests/bench and the oracle.

This module holds NO arithmetic of the method (no predicate evaluation, no
distances, no selection): it only draws the corpus, attributes, queries and
predicate bounds of the five BASELINE.json configurations (recipes in
DESIGN.md "Input recipe").  The paper's own
workloads are synthetic, uniform, seeded ("same random number
generator seed for reproducibility ... generated uniformly at random"), so
no public suite is stood in for.

Reproducibility: every value is a function of (seed, stream, chunk) where a
chunk is CHUNK consecutive global rows, so any row range -- a GPU shard, a
host-side oracle slice -- regenerates identically on the same device type.
CPU and CUDA torch generators produce different streams; a test always draws
on one device and copies to the other.
"""
from __future__ import annotations

import dataclasses
import math

import torch

CHUNK = 65536
INT32_MIN = -(2 ** 31)

# streams
S_VECTORS, S_ATTR0, S_ATTR1, S_QUERIES, S_CENTROIDS, S_CLUSTER, S_NOISE, S_QCLUSTER = range(8)

L2, IP, COS = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    seed: int
    n: int
    d: int
    metric: int
    k: int
    qs: tuple
    sels: tuple          # target selectivities (fractions)
    kind: str            # "gauss" | "gauss_norm" | "mixture"
    attrs: tuple         # per attribute: ("i32", modulus) or ("u8", modulus)
    gpus: tuple = (1,)
    shard_rows: int = 0  # > 0: weak scaling, each GPU holds this many rows (C4: 50M / 8; C5: 20M / 8)


CONFIGS = {
    "c1": Config("c1", 1, 10_000, 128, L2, 10, (8,), (0.10,), "gauss", (("i32", 1000),)),
    "c2": Config("c2", 2, 1_000_000, 128, IP, 10, (1, 16, 256, 4096), (0.001, 0.01, 0.10, 1.0),
                 "gauss_norm", (("i32", 10_000),), (1, 2, 4, 8)),
    "c3": Config("c3", 3, 10_000_000, 768, L2, 100, (1, 64, 1024),
                 (0.0001, 0.001, 0.01, 0.015625, 0.10, 1.0), "gauss",
                 (("i32", 1 << 20), ("u8", 64)), (1, 2)),
    "c4": Config("c4", 4, 50_000_000, 1536, IP, 100, (1, 256, 8192), (0.001, 0.05, 0.50), "gauss",
                 (("i32", 1_000_000),), (1, 2, 4, 8), 6_250_000),
    "c5": Config("c5", 5, 20_000_000, 256, COS, 50, (2048,), (0.001, 0.01, 0.10, 0.30), "mixture",
                 (("i32", 1031),), (8,), 2_500_000),
}

C5_CENTROIDS = 1024
C5_SIGMA = 0.1


def _gen(device, seed: int, stream: int, chunk: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(((seed * 1_000_003 + stream) * 1_000_033 + chunk) % (2 ** 62))
    return g


def _chunks(r0: int, r1: int):
    c = r0 // CHUNK
    while c * CHUNK < r1:
        a, b = c * CHUNK, (c + 1) * CHUNK
        yield c, max(a, r0), min(b, r1), a
        c += 1


def _fill_rows(out: torch.Tensor, r0: int, r1: int, cols: int, seed: int, stream: int, draw):
    """out[(r - r0)] for r in [r0, r1) from per-chunk generators; draw(g, rows, cols) -> tensor."""
    dev = out.device
    for c, a, b, base in _chunks(r0, r1):
        g = _gen(dev, seed, stream, c)
        full = draw(g, CHUNK, cols)            # always the whole chunk -> shard independent
        out[a - r0:b - r0] = full[a - base:b - base].reshape(out[a - r0:b - r0].shape)


def _randn(dev):
    return lambda g, r, c: torch.randn(r, c, generator=g, device=dev, dtype=torch.float32)


def _randint(dev, m, dtype):
    return lambda g, r, c: torch.randint(0, m, (r, c), generator=g, device=dev,
                                         dtype=torch.int64).to(dtype)


def centroids(cfg: Config, device="cpu") -> torch.Tensor:
    g = _gen(device, cfg.seed, S_CENTROIDS, 0)
    return torch.randn(C5_CENTROIDS, cfg.d, generator=g, device=device, dtype=torch.float32)


def rows_of(cfg: Config, world: int, rank: int):
    """(r0, r1, n_total) of `rank`'s shard: weak scaling (shard_rows per GPU, the
    first `world` shards of the global corpus) when the config has shard_rows,
    else the contiguous 1/world of cfg.n (strong scaling)."""
    if cfg.shard_rows:
        return rank * cfg.shard_rows, (rank + 1) * cfg.shard_rows, cfg.shard_rows * world
    return cfg.n * rank // world, cfg.n * (rank + 1) // world, cfg.n


def corpus(cfg: Config, r0: int = 0, r1: int | None = None, device="cpu", n: int | None = None,
           d: int | None = None):
    """Rows [r0, r1) of the corpus: (X fp32 [m, d] row-major, [attr columns]).

    n / d override the config's sizes (parity tests at reduced sizes keep the
    distributions and the predicate structure)."""
    n = cfg.n if n is None else n
    d = cfg.d if d is None else d
    r1 = n if r1 is None else r1
    m = r1 - r0
    dev = torch.device(device)
    X = torch.empty(m, d, dtype=torch.float32, device=dev)
    if cfg.kind in ("gauss", "gauss_norm"):
        _fill_rows(X, r0, r1, d, cfg.seed, S_VECTORS, _randn(dev))
        if cfg.kind == "gauss_norm":   # input preparation: rows L2-normalised (BASELINE configs[1])
            X /= X.norm(dim=1, keepdim=True)
    elif cfg.kind == "mixture":        # BASELINE configs[4]: x = c_cid + 0.1 N(0, I)
        cen = centroids(cfg, dev) if d == cfg.d else centroids(dataclasses.replace(cfg, d=d), dev)
        cid = torch.empty(m, 1, dtype=torch.int64, device=dev)
        _fill_rows(cid, r0, r1, 1, cfg.seed, S_CLUSTER, _randint(dev, C5_CENTROIDS, torch.int64))
        _fill_rows(X, r0, r1, d, cfg.seed, S_VECTORS, _randn(dev))
        X.mul_(C5_SIGMA).add_(cen[cid[:, 0]])
    else:
        raise ValueError(cfg.kind)
    attrs = []
    for ai, (typ, mod) in enumerate(cfg.attrs):
        if cfg.kind == "mixture" and ai == 0:   # a0 = cluster id + U{0..7}
            noise = torch.empty(m, 1, dtype=torch.int64, device=dev)
            _fill_rows(noise, r0, r1, 1, cfg.seed, S_NOISE, _randint(dev, 8, torch.int64))
            attrs.append((cid[:, 0] + noise[:, 0]).to(torch.int32))
            continue
        dt = torch.int32 if typ == "i32" else torch.uint8
        col = torch.empty(m, 1, dtype=dt, device=dev)
        _fill_rows(col, r0, r1, 1, cfg.seed, S_ATTR0 + ai, _randint(dev, mod, dt))
        attrs.append(col[:, 0].contiguous())
    return X, attrs


def queries(cfg: Config, q: int, device="cpu", d: int | None = None) -> torch.Tensor:
    """Query batch [q, d]; drawn from the corpus distribution (SURVEY 8(c) reading 13, 22)."""
    d = cfg.d if d is None else d
    dev = torch.device(device)
    g = _gen(dev, cfg.seed, S_QUERIES, 0)
    Qv = torch.randn(q, d, generator=g, device=dev, dtype=torch.float32)
    if cfg.kind == "gauss_norm":
        Qv /= Qv.norm(dim=1, keepdim=True)
    elif cfg.kind == "mixture":
        cen = centroids(dataclasses.replace(cfg, d=d), dev)
        g2 = _gen(dev, cfg.seed, S_QCLUSTER, 0)
        j = torch.randint(0, C5_CENTROIDS, (q,), generator=g2, device=dev)
        Qv = cen[j] + C5_SIGMA * Qv
    return Qv.contiguous()


def predicate(cfg: Config, sel: float):
    """Clauses [(attr, lo, hi)] (AND of closed intervals) whose expected
    selectivity is `sel` on this config's attribute distributions."""
    if cfg.name == "c1":
        return [(0, INT32_MIN, round(sel * 1000) - 1)]            # attr < 100 at 10 %
    if cfg.name in ("c2", "c4"):
        mod = cfg.attrs[0][1]
        return [(0, INT32_MIN, round(sel * mod) - 1)]             # a0 <= s*m - 1
    if cfg.name == "c3":
        T = 1 << 20
        if sel >= 1.0:
            W, C = T, 64
        elif sel <= 1.0 / 64:
            C = 1
            W = min(T, round(sel * T * 64))
        else:
            C = 8 if sel <= 0.125 else 64
            W = min(T, round(sel * T * 64 / C))
        t0 = (T - W) * 37 // 100
        c0 = (64 - C) // 2
        return [(0, t0, t0 + W - 1), (1, c0, c0 + C - 1)]
    if cfg.name == "c5":
        w = max(1, round(sel * 1024))
        w = min(w, 1017)
        a = 7 + (1017 - w) // 2
        return [(0, a, a + w - 1)]
    raise ValueError(cfg.name)


def expected_selectivity(cfg: Config, clauses) -> float:
    """Analytic selectivity of `clauses` under the attribute distributions."""
    if cfg.name == "c5":
        (a, lo, hi), = clauses
        # a0 = cid + u, cid ~ U{0..1023}, u ~ U{0..7}: P(lo <= a0 <= hi)
        p = 0.0
        for v in range(lo, hi + 1):
            cnt = sum(1 for u in range(8) if 0 <= v - u < C5_CENTROIDS)
            p += cnt / (C5_CENTROIDS * 8)
        return p
    p = 1.0
    for (a, lo, hi) in clauses:
        mod = cfg.attrs[a][1]
        lo_c, hi_c = max(lo, 0), min(hi, mod - 1)
        p *= max(0, hi_c - lo_c + 1) / mod
    return p


def seeded_rng(seed: int):
    """Small-case generator for tests (numpy)."""
    import numpy as np
    return np.random.default_rng(seed)


def round_up(x: int, m: int) -> int:
    return int(math.ceil(x / m) * m)
