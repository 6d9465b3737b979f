#!/usr/bin/env python
"""bench.py -- filtered exact top-k queries/sec on B200 (BASELINE.json metric).

One STEP = one pass of the whole hot path over every (selectivity, Q) cell of
the workload.  Default: configs[3] = "c4", the configuration BASELINE's metric
is quoted on ("at 1/2/4/8 B200"): N = 50M fp32 d = 1536 rows, IP, k = 100,
s in {0.1, 5, 50} %, Q in {1, 256, 8192}; weak scaling -- rank r holds the
6.25M-row shard r, so N GPUs search the first N shards (8 GPUs = the full
50M corpus).  Per cell one vrs_search (predicate -> selection -> distances ->
fused top-k -> exact re-score -> certificate, exact fallback if needed); on
N > 1 GPUs one NCCL all-gather of the step's per-shard [Q x k] candidates and
one vrs_merge.  value = queries answered per second by the whole job (every
answer the exact top-k over the corpus the job holds).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4] [--impl ours|reference]

--gpus N > 1 without torchrun's environment relaunches itself under
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402

METRIC = "filtered exact top-k queries/sec and % of HBM/tensor roofline at 1/2/4/8 B200"
UNIT = "queries/s"
NOMINAL_TF32_OVER_BF16 = 1.1 / 2.25   # B200_PROFILING.md nominal dense tf32 / bf16 (fp16 = bf16)


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    return p


def host_info():
    model, mem = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                mem = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "ram_gib": mem, "cores_visible": len(os.sched_getaffinity(0))}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.lines, self.proc = dev, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float):
        """Block until the first sample arrived (or timeout): starting nvidia-smi initialises
        NVML, which can stall the GPU for tens of ms -- that must not land in a timed step."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)
        time.sleep(0.05)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons), "samples": len(sm)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a captured CUDA graph")
    ap.add_argument("--no-cells", action="store_true", help="skip the per-cell timing table")
    ap.add_argument("--precision", default=None, choices=["tf32", "bf16", "fp16"],
                    help="selection operand precision of the index (default: the library's, fp16)")
    return ap.parse_args()


def relaunch_distributed(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run (N ranks)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def cells_of(cfg):
    return [(s, q) for s in cfg.sels for q in cfg.qs]


def workload_desc(cfg, world):
    r0, r1, n_tot = datagen.rows_of(cfg, world, 0)
    return {"workload": f"{cfg.name} (BASELINE.json configs[{list(datagen.CONFIGS).index(cfg.name)}])",
            "n": n_tot, "d": cfg.d, "metric": ["l2", "ip", "cos"][cfg.metric], "k": cfg.k,
            "rows_per_gpu": r1 - r0,
            "sharding": ("weak: rank r holds shard r of %d rows; N GPUs search the first N shards" % cfg.shard_rows
                         if cfg.shard_rows else "strong: the corpus split contiguously over the GPUs"),
            "selectivities": list(cfg.sels), "queries_per_cell": list(cfg.qs), "cells": len(cells_of(cfg)),
            "queries_per_step": sum(q for _, q in cells_of(cfg)),
            "data": "synthetic, seeded (datagen): BASELINE.json configs shapes and distributions",
            "l2_flush": "inputs > L2 (corpus %.1f GB fp32 + %.1f GB fp16 shadow per GPU vs 126 MB L2)" % (
                (r1 - r0) * cfg.d * 4 / 1e9, (r1 - r0) * cfg.d * 2 / 1e9),
            "parallelism": (f"{world} GPUs, rows sharded, one exchange + merge of the step's candidates (vrs_merge_push over symmetric memory, else NCCL all-gather + vrs_merge)"
                            if world > 1 else "1 GPU")}


# --------------------------------------------------------------------------- oracle legs
def _oracle_slice(cfg, rank_rows, dev, max_rows):
    """A bounded host slice of the shard for the CPU oracle: rows [r0, r0 + m)."""
    r0, r1 = rank_rows
    m = min(r1 - r0, max_rows)
    X, attrs = datagen.corpus(cfg, r0, r0 + m, dev)
    return X.cpu().numpy(), [a.cpu().numpy() for a in attrs], m


def oracle_sample(cfg, X_h, attrs_h, rows_total, Q_h, per_sel_queries: int, threads: int):
    """Time the CPU oracle on `per_sel_queries` queries per selectivity over the host
    slice X_h (the first rows of the shard) and extrapolate linearly to the shard's
    rows_total rows and to the step's query mix.  Returns (qps, seconds, desc)."""
    import oracle
    tq = {}
    t_all = 0.0
    scale = rows_total / X_h.shape[0]
    for s in cfg.sels:
        pred = datagen.predicate(cfg, s)
        t0 = time.perf_counter()
        oracle.search(X_h, attrs_h, pred, Q_h[:per_sel_queries], cfg.k, cfg.metric, 0, threads)
        dt = time.perf_counter() - t0
        t_all += dt
        tq[s] = dt / per_sel_queries * scale
    total_q = sum(q for _, q in cells_of(cfg))
    total_t = sum(q * tq[s] for s, q in cells_of(cfg))
    desc = (f"{per_sel_queries} queries x {len(cfg.sels)} selectivities over the first {X_h.shape[0]} rows of the "
            f"{rows_total}-row shard (oracle: fp64 brute force + sort, {threads} threads); per-query time scaled "
            f"x{scale:.2f} to the shard and extrapolated to the step's {total_q} queries")
    return total_q / total_t, t_all, desc


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    import oracle
    oracle.build()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))) if torch.cuda.is_available() else "cpu"
    r0, r1, _ = datagen.rows_of(cfg, 1, 0)
    X_h, attrs_h, m = _oracle_slice(cfg, (r0, r1), dev, 1_000_000)
    Q_h = datagen.queries(cfg, 64, dev).cpu().numpy()
    threads = len(os.sched_getaffinity(0))
    per = 1
    for _ in range(args.warmup):
        oracle_sample(cfg, X_h, attrs_h, r1 - r0, Q_h, per, threads)
    times, qps = [], []
    for _ in range(args.steps):
        v, t, desc = oracle_sample(cfg, X_h, attrs_h, r1 - r0, Q_h, per, threads)
        times.append(t)
        qps.append(v)
    value = statistics.median(qps)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak" if cfg.shard_rows else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_desc(cfg, 1),
            "cpu_baseline": dict(value=value, unit=UNIT, cores=threads, kind="oracle", sample=desc, **host_info()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def oracle_topk_shard(cfg, X_dev, attrs_dev, pred, Q_h, row_offset, threads=0):
    """Oracle top-k of Q_h over one (GPU-resident) shard, reading only the rows the
    ORACLE's own selection keeps: attributes -> host -> oracle.select -> those rows
    copied to the host (torch indexing: plumbing) -> oracle.search over them with the
    empty predicate; local positions map back through the oracle's ascending ids, so the
    id tie-break is unchanged.  -> (ids int64 [q, k] global, dists f32 [q, k])."""
    import oracle
    attrs_h = [a.cpu().numpy() for a in attrs_dev]
    n = X_dev.shape[0]
    _, cnt, sel = oracle.select(attrs_h, n, pred)
    k = cfg.k
    ids = np.full((Q_h.shape[0], k), -1, dtype=np.int64)
    dists = np.full((Q_h.shape[0], k), np.inf if cfg.metric == datagen.L2 else -np.inf, dtype=np.float32)
    if cnt == 0:
        return ids, dists
    parts_i, parts_d = [], []
    step = 400_000
    for c0 in range(0, cnt, step):   # bounded host memory: the selection in chunks, merged by the oracle
        sl = sel[c0:c0 + step]
        Xs = X_dev.index_select(0, torch.from_numpy(sl).to(X_dev.device)).cpu().numpy()
        li, ld, _ = oracle.search(Xs, [], [], Q_h, k, cfg.metric, 0, threads)
        gi = np.where(li >= 0, sl[np.clip(li, 0, None)] + row_offset, -1)
        parts_i.append(gi)
        parts_d.append(ld)
    if len(parts_i) == 1:
        return parts_i[0], parts_d[0]
    return oracle.merge(np.stack(parts_i), np.stack(parts_d), k, cfg.metric)


def compare_exact(gi, gd, ri, rd):
    """Certified-exact contract: ids rank for rank, dists within one fp32 ulp."""
    bad_ids = int((gi != ri).any(axis=1).sum())
    ulp = np.spacing(np.abs(rd).astype(np.float32))
    fin = np.isfinite(rd)
    bad_d = int(((np.abs(gd.astype(np.float64) - rd.astype(np.float64)) > ulp) & fin).any(axis=1).sum())
    return bad_ids, bad_d


# --------------------------------------------------------------------------- our path
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    cfg = datagen.CONFIGS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}")
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import paper_2403_15807_b200 as vrs
    vrs.library()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    r0, r1, n_total = datagen.rows_of(cfg, world, rank)
    X, attrs = datagen.corpus(cfg, r0, r1, dev)
    qmax = max(cfg.qs)
    Qall = datagen.queries(cfg, qmax, dev)
    prec = {None: None, "tf32": vrs.PREC_TF32, "bf16": vrs.PREC_BF16, "fp16": vrs.PREC_FP16}[args.precision]
    ix = vrs.Index(X, attrs, row_offset=r0, precision=prec)
    cells = cells_of(cfg)
    preds = {s: datagen.predicate(cfg, s) for s in cfg.sels}
    k, metric = cfg.k, cfg.metric
    # every cell's local results are views of two step-wide buffers, so that N > 1 merges
    # the whole step with ONE all-gather per array and ONE vrs_merge (not one per cell)
    q_tot = sum(q for _, q in cells)
    ids_all = torch.empty(q_tot, k, dtype=torch.int64, device=dev)
    dists_all = torch.empty(q_tot, k, dtype=torch.float32, device=dev)
    bufs, q0 = {}, 0
    offs = {}
    for c in cells:
        bufs[c] = (ids_all[q0:q0 + c[1]], dists_all[q0:q0 + c[1]])
        offs[c] = q0
        q0 += c[1]
    merge_path = None
    if world > 1:
        import torch.distributed as dist
        from paper_2403_15807_b200.dist import PeerMerge, gather_merge
        # the exchange + merge as one kernel over symmetric (NVLink peer) memory; NCCL
        # all-gather + vrs_merge when symmetric memory is unavailable
        nccl_path = "NCCL all_gather_into_tensor + vrs_merge"
        try:
            peer = PeerMerge(q_tot, k)
            merge_path = "vrs_merge_push: one kernel, P2P pushes into torch symmetric memory + device-side wait + merge"
        except Exception as e:   # noqa: BLE001 -- fall back to the collective
            peer = None
            merge_path = f"{nccl_path} (symmetric memory unavailable: {type(e).__name__})"
        # every rank must take the same path: the push kernel only if every rank built it AND one
        # validation exchange equals the NCCL path's result on every rank with no expired wait
        # (the kernel's wait is bounded, vrs.h: a transport that does not deliver cannot hang the run)
        have = torch.tensor([1 if peer is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(have, op=dist.ReduceOp.MIN)
        if peer is not None and not have.item():
            peer, merge_path = None, f"{nccl_path} (symmetric memory unavailable on another rank)"
        if peer is not None and not peer.validate(metric):
            peer, merge_path = None, f"{nccl_path} (vrs_merge_push failed its validation exchange against the NCCL path)"

        def exchange(ids_t, dists_t):
            if peer is not None and ids_t.shape[0] == q_tot:
                return peer.merge(ids_t, dists_t, metric)
            return gather_merge(ids_t, dists_t, k, metric)
    launches = [0]
    merged = [None]
    cell_path = {}

    def run_cell(c, stats=None):
        s, q = c
        ids, dists = ix.search(Qall[:q], preds[s], k=k, metric=metric, out=bufs[c], stats=stats)
        launches[0] += vrs.last_launches()
        cell_path[c] = vrs.last_path()
        return ids, dists

    def step(stats=None):
        for c in cells:
            run_cell(c, stats)
        if world > 1:   # the step's results: one push-merge kernel (or all-gather + vrs_merge)
            merged[0] = exchange(ids_all, dists_all)
            launches[0] += 1

    def barrier():
        if world > 1:
            dist.barrier()

    # selection sizes (outside timing) for the algorithmic byte / flop counts
    nsel = {}
    for s in cfg.sels:
        _, cnt, _ = ix.select(preds[s])
        nsel[s] = int(cnt.item())

    # certificate statistics over one (untimed) step: queries, uncertified (exact fallback), bound check
    cst = vrs.new_stats(dev)
    step(cst)
    torch.cuda.synchronize()
    cert = vrs.read_stats(cst)

    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first(5.0)   # nvidia-smi's NVML start-up done before anything is timed
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    # the step (every cell's launches, scratch allocation, and on N > 1 the NCCL all-gather
    # + merge) is captured once as a CUDA graph and replayed, so small cells measure the
    # GPU rather than Python's launch loop; eager launches if capture is refused
    graph, timing = None, "eager launches"
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            launches[0] = 0
            with torch.cuda.graph(graph, stream=cap):
                step()
            launches_per_step = launches[0]
            graph.replay()
            torch.cuda.synchronize()
            barrier()
            timing = ("CUDA graph of the step (captured once, outside the timed region"
                      + (", the exchange + merge inside" if world > 1 else "") + "), replayed K times")
        except Exception as e:   # noqa: BLE001 -- report and time eagerly
            graph = None
            timing = f"eager launches (graph capture failed: {type(e).__name__})"
            torch.cuda.synchronize()
            barrier()

    # ---------------- timed region
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e0.record(stream)
    for i in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
        step_ev[i].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    step_ms = [e0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i]) for i in range(1, args.steps)]
    gpu_launches = launches_per_step * args.steps if graph is not None else launches[0]
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    q_per_step = sum(q for _, q in cells)
    value = args.steps * q_per_step / (ms / 1e3)

    # ---------------- per-kernel CUDA-event pass (same steps) -> roofline of the dominant kernel
    vrs.profile(True)
    vrs.profile_reset()
    nprof = min(args.steps, 3)
    for _ in range(nprof):
        step()
    torch.cuda.synchronize()
    prof = vrs.profile_read()
    vrs.profile(False)
    pk = peaks()
    h16 = ix.precision in (vrs.PREC_BF16, vrs.PREC_FP16)
    d = cfg.d
    n_loc = r1 - r0
    flops_gemm = bytes_scan = 0.0
    for s, q in cells:
        ns = nsel[s]
        if cell_path[(s, q)] == vrs.PATH_GEMM:
            flops_gemm += 2.0 * q * ns * d
        else:
            bytes_scan += ns * (4.0 * d + 12) + q * 4.0 * d
    step_s = ms / args.steps / 1e3
    flat = {kname: v for kname, v in prof.items() if kname != "gemm"}
    dominant = "gemm.main" if "gemm.main" in flat else (max(flat.items(), key=lambda kv: kv[1][0])[0] if flat else None)
    roof = None
    if dominant == "gemm.main":
        t_s = prof["gemm.main"][0] / 1e3 / nprof
        ach = flops_gemm / t_s / 1e12
        # burst peak for a pass timed inside a step of < ~1 s, the sustained one for steps of seconds
        burst = step_s < 1.0
        if h16:   # kind::f16 (fp16 shadow): the measured bf16 peak (fp16 = bf16 nominal rate)
            peak = pk["bf16_tflops"] if burst else pk["bf16_tflops_sustained"]
            kind, note = "fp16" if ix.precision == vrs.PREC_FP16 else "bf16", "measured bf16 cuBLAS peak (fp16 dense = bf16 nominal)"
        else:
            peak = (pk["bf16_tflops"] if burst else pk["bf16_tflops_sustained"]) * NOMINAL_TF32_OVER_BF16
            kind, note = "TF32", "measured bf16 peak x nominal tf32/bf16 (1.1/2.25)"
        roof = {"kernel": f"tc_topk_kernel main pass (tcgen05 kind::f16 {kind} + fused top-k)", "bound": "tensor",
                "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "traffic": None,
                "peak_note": note + (": burst (step %.0f ms)" % (step_s * 1e3) if burst else ": sustained"),
                "algorithmic": "2*Q*N_sel*d per tensor-core cell, summed over the step, / the step's main-pass time "
                               "(CUDA events on the launch stream)"}
        tr = os.path.join(ROOT, "profiles", f"r02_ncu_{cfg.name}_main_traffic.json")
        if os.path.exists(tr):
            tj = json.load(open(tr))
            roof["traffic"] = tj.get("dram_bytes_per_launch")
            roof["traffic_evidence"] = tj.get("what")
            roof["traffic_algorithmic_bytes"] = tj.get("algorithmic_bytes")
    elif dominant is not None:
        t_s = prof[dominant][0] / 1e3 / nprof
        ach = bytes_scan / t_s / 1e9
        roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach / pk["hbm_gbs"], "traffic": None,
                "algorithmic": "N_sel*(4d+12) + 4*Q*d bytes per scan cell"}
    if roof is not None:
        roof["peak_source"] = pk["source"]
        roof["kernel_share_of_step"] = {kname: v[0] / nprof / (ms / args.steps) for kname, v in prof.items()}

    # ---------------- per-cell timings (events around each cell)
    cell_out = []
    if not args.no_cells:
        for c in cells:
            s, q = c
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            run_cell(c)
            torch.cuda.synchronize()
            # the cell alone as a CUDA graph (device time; eager launches of a tiny cell would
            # time Python's launch loop), replayed `reps` times between two events
            cg = None
            if graph is not None:
                try:
                    cap_c = torch.cuda.Stream()
                    cap_c.wait_stream(torch.cuda.current_stream())
                    cg = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(cg, stream=cap_c):
                        run_cell(c)
                    cg.replay()
                    torch.cuda.synchronize()
                except Exception:   # noqa: BLE001 -- eager timing instead
                    cg = None
                    torch.cuda.synchronize()
            reps = 5 if cg is not None else 3
            a.record(stream)
            for _ in range(reps):
                if cg is not None:
                    cg.replay()
                else:
                    run_cell(c)
            b.record(stream)
            torch.cuda.synchronize()
            del cg
            t = a.elapsed_time(b) / reps / 1e3
            ns = nsel[s]
            fl = 2.0 * q * ns * d
            esz = 2.0 if (vrs.last_path() == vrs.PATH_GEMM and h16) else 4.0
            by = n_loc * sum(1 if cfg.attrs[i][0] == "u8" else 4 for i in range(len(cfg.attrs))) + ns * esz * d \
                + q * 4.0 * d + q * k * 12
            tc_peak = pk["bf16_tflops"] * (1.0 if h16 else NOMINAL_TF32_OVER_BF16)
            path = "gemm" if vrs.last_path() == vrs.PATH_GEMM else "scan"
            # the cell's kernel split: one more call with per-kernel CUDA events (ProfScope)
            vrs.profile(True)
            vrs.profile_reset()
            run_cell(c)
            torch.cuda.synchronize()
            kms = {kname: round(v[0], 4) for kname, v in vrs.profile_read().items()}
            vrs.profile(False)
            hf, tf = by / t / 1e9 / pk["hbm_gbs"], fl / t / 1e12 / tc_peak
            cell_out.append({"sel": s, "q": q, "n_sel": ns, "ms": t * 1e3, "qps": q / t, "path": path,
                             "timing": "graph replay" if reps == 5 else "eager",
                             "hbm_frac": hf, "tensor_frac_burst": tf,
                             "binding": "tensor" if fl / (tc_peak * 1e12) > by / (pk["hbm_gbs"] * 1e9) else "hbm",
                             "kernels_ms": kms})

    # ---------------- e2e through the public API with host buffers
    h2d = sum(q * d * 4 for _, q in cells)
    d2h = sum(q * k * 12 for _, q in cells)
    Qh = Qall.cpu().pin_memory()
    nbuf = 2
    hbufs = [{c: (torch.empty(c[1], k, dtype=torch.int64, pin_memory=True),
                  torch.empty(c[1], k, dtype=torch.float32, pin_memory=True)) for c in cells} for _ in range(nbuf)]
    qh = {q: Qh[:q].clone().pin_memory() for q in cfg.qs}
    step_done = [torch.cuda.Event() for _ in range(nbuf)]
    e2e_i = [0]
    if world > 1:
        qd = {q: torch.empty(q, d, device=dev) for q in cfg.qs}

    def e2e_step():
        slot = e2e_i[0] % nbuf
        e2e_i[0] += 1
        step_done[slot].synchronize()   # the results of the step that last used this set are in host memory
        hb = hbufs[slot]
        for c in cells:
            s, q = c
            if world == 1:
                # the public host-buffer call: queries H2D, search, ids / dists D2H (host_async)
                ix.search_host(qh[q], preds[s], k=k, metric=metric, out=hb[c], host_async=2)
            else:
                qd[q].copy_(qh[q], non_blocking=True)
                ix.search(qd[q], preds[s], k=k, metric=metric, out=bufs[c])
        if world > 1:   # one exchange + merge for the step, results to the host
            mi, md = exchange(ids_all, dists_all)
            for c in cells:
                hb[c][0].copy_(mi[offs[c]:offs[c] + c[1]], non_blocking=True)
                hb[c][1].copy_(md[offs[c]:offs[c] + c[1]], non_blocking=True)
        if world == 1:
            ix.host_fence(stream)   # the step's event covers every result download
        step_done[slot].record(stream)

    e2e_step()
    torch.cuda.synchronize()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    ems = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ems], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e = {"value": args.steps * q_per_step / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "pipelining": "2 pinned result sets; the host waits on a step's event before reusing its set; "
                         "downloads overlap the next cell's kernels (host_async = 2, vrs_host_fence per step)"}

    # ---------------- sampled parity at full size (every rank: its shard's oracle; rank 0 merges)
    parity = None
    if not args.no_parity:
        import oracle
        oracle.build()
        nq = 3 if world == 1 else 2
        Q_h = Qall[:nq].cpu().numpy()
        # (the oracle reads the selection in bounded chunks; at N > 1 the ranks share the host's
        # cores, so the largest selectivity is left to the N = 1 run)
        pcells = [(s, max(cfg.qs)) for s in (cfg.sels if world == 1 else cfg.sels[:-1])]
        res = []
        for s, q in pcells:
            run_cell((s, q))
            torch.cuda.synchronize()
            if world > 1:   # the merged result of this cell (every rank runs the same merge)
                gi_t, gd_t = gather_merge(*bufs[(s, q)], k, metric)
            else:
                gi_t, gd_t = bufs[(s, q)]
            gi, gd = gi_t[:nq].cpu().numpy(), gd_t[:nq].cpu().numpy()
            ri, rd = oracle_topk_shard(cfg, X, attrs, preds[s], Q_h, r0, max(1, len(os.sched_getaffinity(0)) // world))
            if world > 1:   # gather every rank's oracle top-k, merge with the oracle's merge
                ti = torch.from_numpy(ri).to(dev)
                td = torch.from_numpy(rd).to(dev)
                ai = [torch.empty_like(ti) for _ in range(world)]
                ad = [torch.empty_like(td) for _ in range(world)]
                dist.all_gather(ai, ti)
                dist.all_gather(ad, td)
                ri, rd = oracle.merge(np.stack([x.cpu().numpy() for x in ai]), np.stack([x.cpu().numpy() for x in ad]),
                                      k, cfg.metric)
            bi, bd = compare_exact(gi, gd, ri, rd)
            res.append({"sel": s, "q_cell": q, "queries_checked": nq, "bad_id_rows": bi, "bad_dist_rows": bd})
        # A1 / A2 in full for every selectivity: bitmap words and count bit-exact vs the oracle's selection
        bm_ok = True
        for s in cfg.sels:
            bm, cnt, _ = ix.select(preds[s])
            obm, ocnt, _ = oracle.select([a.cpu().numpy() for a in attrs], n_loc, preds[s])
            gbm = bm.cpu().numpy().view(np.uint32)
            bm_ok &= int(cnt.item()) == ocnt and np.array_equal(gbm, obm[: gbm.size])
        ok = bm_ok and all(r["bad_id_rows"] == 0 and r["bad_dist_rows"] == 0 for r in res)
        parity = {"cells": res, "bitmaps_bit_exact": bool(bm_ok), "ok": bool(ok),
                  "rule": "certified exact (DESIGN.md Sec. 7): ids identical to the oracle's rank for rank, dists "
                          "within one fp32 ulp of fp32(oracle fp64); bitmap + count bit-exact for every selectivity",
                  "oracle": ("per rank: its shard's oracle top-k over the oracle's own selection; rank 0 merges them "
                             "with oracle.merge" if world > 1 else "the shard's oracle top-k over the oracle's own selection")}
        if not ok:
            print("PARITY FAILURE: " + json.dumps(parity), file=sys.stderr, flush=True)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        X_h, attrs_h, _ = _oracle_slice(cfg, (r0, r1), dev, 1_000_000)
        v, t_all, desc = oracle_sample(cfg, X_h, attrs_h, r1 - r0, Qall[:4].cpu().numpy(), 2, threads)
        cpu = dict(value=v, unit=UNIT, cores=threads, kind="oracle", sample=desc, sample_seconds=t_all, **host_info())

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak" if cfg.shard_rows else "strong", "vs_baseline": None,
                "dtype": {vrs.PREC_FP16: "fp16", vrs.PREC_BF16: "bf16"}.get(ix.precision, "tf32"),
                "dtype_note": "tensor-core selection operands (fp32 accumulate); every result re-scored in fp64 "
                              "from fp32 and certified exact (uncertified queries recomputed in fp64)",
                "data": "synthetic", "config": workload_desc(cfg, world), "e2e": e2e,
                "gpu_launches": gpu_launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
                "timing": timing, "certificate": cert, "parity": parity, "cells": cell_out,
                "merge": merge_path,
                "merge_wait_expired": (bool(peer.timed_out()) if world > 1 and peer is not None else None),
                "step_ms": [round(x, 4) for x in step_ms],
                "kernels_ms_per_step": {kname: v[0] / nprof for kname, v in prof.items()}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
