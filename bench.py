#!/usr/bin/env python
"""bench.py -- filtered exact top-k queries/sec on B200 (BASELINE.json metric).

One STEP = one pass of the whole hot path over every (selectivity, Q) cell of
the workload (default configs[1] = "c2": N=1M fp32 d=128 L2-normalised, IP,
s in {0.1,1,10,100} %, Q in {1,16,256,4096}, k=10): per cell one
vrs_search (predicate -> selection -> distances -> fused top-k -> exact
re-score), plus, on N > 1 GPUs, an NCCL all-gather of the per-shard [Q x k]
candidates and vrs_merge.  value = queries answered per second by the whole
job (all cells, all ranks' shards merged).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

Multi-GPU: launched by torchrun, one process per GPU; the corpus rows are
sharded contiguously over the ranks (strong scaling of the workload's N).
"""
from __future__ import annotations

import argparse
import json
import os
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
NOMINAL_TF32_OVER_BF16 = 1.1 / 2.25   # B200_PROFILING.md nominal dense tf32 / bf16


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured"
    return p


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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of replaying the step's captured CUDA graph (N = 1)")
    return ap.parse_args()


def cells_of(cfg):
    return [(s, q) for s in cfg.sels for q in cfg.qs]


def workload_desc(cfg, world):
    return {"workload": f"{cfg.name} (BASELINE.json configs[{list(datagen.CONFIGS).index(cfg.name)}])",
            "n": datagen.rows_of(cfg, world, 0)[2], "d": cfg.d, "metric": ["l2", "ip", "cos"][cfg.metric],
            "k": cfg.k, "rows_per_gpu": datagen.rows_of(cfg, world, 0)[1],
            "selectivities": list(cfg.sels), "queries_per_cell": list(cfg.qs), "cells": len(cells_of(cfg)),
            "data": "synthetic, seeded (datagen)", "l2_flush": "inputs > L2 (corpus %.0f MB per GPU)" % (datagen.rows_of(cfg, world, 0)[1] * cfg.d * 4 / 1e6),
            "parallelism": f"rows sharded over {world} GPU(s), one NCCL all-gather per step + merge" if world > 1 else "1 GPU"}


# --------------------------------------------------------------------------- oracle legs
def oracle_sample(cfg, X_h, attrs_h, Q_h, per_sel_queries: int, threads: int):
    """Time the CPU oracle on `per_sel_queries` queries per selectivity over the full
    (local) corpus; extrapolate to the step's query mix.  Returns (qps, seconds, desc)."""
    import oracle
    tq = {}
    t_all = 0.0
    for s in cfg.sels:
        pred = datagen.predicate(cfg, s)
        t0 = time.perf_counter()
        oracle.search(X_h, attrs_h, pred, Q_h[:per_sel_queries], cfg.k, cfg.metric, 0, threads)
        dt = time.perf_counter() - t0
        t_all += dt
        tq[s] = dt / per_sel_queries
    total_q = sum(q for _, q in cells_of(cfg))
    total_t = sum(q * tq[s] for s, q in cells_of(cfg))
    desc = (f"{per_sel_queries} queries x {len(cfg.sels)} selectivities over the full {X_h.shape[0]}-row corpus "
            f"(oracle: fp64 brute force + sort), per-query time extrapolated to the step's {total_q} queries")
    return total_q / total_t, t_all, desc, total_t


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    import oracle
    oracle.build()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))) if torch.cuda.is_available() else "cpu"
    r0, r1, _ = datagen.rows_of(cfg, 1, 0)
    X, attrs = datagen.corpus(cfg, r0, r1, dev)
    Q = datagen.queries(cfg, 64, dev)
    X_h, attrs_h, Q_h = X.cpu().numpy(), [a.cpu().numpy() for a in attrs], Q.cpu().numpy()
    del X
    threads = len(os.sched_getaffinity(0))
    per = 1
    for _ in range(args.warmup):
        oracle_sample(cfg, X_h, attrs_h, Q_h, per, threads)
    times, qps = [], []
    for _ in range(args.steps):
        v, t, desc, _ = oracle_sample(cfg, X_h, attrs_h, Q_h, per, threads)
        times.append(t)
        qps.append(v)
    value = statistics.median(qps)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak" if cfg.shard_rows else "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic", "config": workload_desc(cfg, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our path
def main():
    args = parse()
    cfg = datagen.CONFIGS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    ix = vrs.Index(X, attrs, row_offset=r0)
    cells = cells_of(cfg)
    preds = {s: datagen.predicate(cfg, s) for s in cfg.sels}
    k, metric = cfg.k, cfg.metric
    # every cell's local results are views of two step-wide buffers, so that N > 1 merges
    # the whole step with ONE all-gather per array and ONE vrs_merge (not one per cell)
    q_tot = sum(q for _, q in cells)
    ids_all = torch.empty(q_tot, k, dtype=torch.int64, device=dev)
    dists_all = torch.empty(q_tot, k, dtype=torch.float32, device=dev)
    bufs, q0 = {}, 0
    for c in cells:
        bufs[c] = (ids_all[q0:q0 + c[1]], dists_all[q0:q0 + c[1]])
        q0 += c[1]
    if world > 1:
        import torch.distributed as dist
        from paper_2403_15807_b200.dist import gather_merge
    launches = [0]

    cell_path = {}

    def run_cell(c, merge=True):
        s, q = c
        ids, dists = ix.search(Qall[:q], preds[s], k=k, metric=metric, out=bufs[c])
        launches[0] += vrs.last_launches()
        cell_path[c] = vrs.last_path()
        if world > 1 and merge:
            out = gather_merge(ids, dists, k, metric)   # NCCL all-gather + vrs_merge
            launches[0] += 1
            return out
        return ids, dists

    def step():
        for c in cells:
            run_cell(c, merge=False)
        if world > 1:   # the step's results: one NCCL all-gather per array + one vrs_merge
            gather_merge(ids_all, dists_all, k, metric)
            launches[0] += 1

    def barrier():
        if world > 1:
            dist.barrier()

    # selection sizes (outside timing) for the algorithmic byte / flop counts
    nsel = {}
    for s in cfg.sels:
        _, cnt, _ = ix.select(preds[s])
        nsel[s] = int(cnt.item())

    # clock sampler first, then the warm-up: the timed steps follow the warm-up
    # without an idle gap (an idle GPU drops its clocks; the first timed step
    # would pay for the ramp)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first(5.0)   # nvidia-smi's NVML start-up done before anything is timed
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    # N = 1: the step (every cell's launches, scratch allocation included) is captured
    # once as a CUDA graph and replayed, so tiny configs measure the GPU, not Python's
    # launch loop (C1: ~40 us of host time per call against ~40 us of kernels)
    graph = None
    if world == 1 and not args.no_graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        launches[0] = 0
        with torch.cuda.graph(graph, stream=cap):
            step()
        launches_per_step = launches[0]
        graph.replay()
        torch.cuda.synchronize()

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
    for _ in range(min(args.steps, 5)):
        step()
    torch.cuda.synchronize()
    prof = vrs.profile_read()
    vrs.profile(False)
    nprof = min(args.steps, 5)
    pk = peaks()
    tf32_peak_sus = pk["bf16_tflops_sustained"] * NOMINAL_TF32_OVER_BF16
    tc_peak_sus = pk["bf16_tflops_sustained"] if ix.precision == vrs.PREC_BF16 else tf32_peak_sus
    tf32_peak_burst = pk["bf16_tflops"] * NOMINAL_TF32_OVER_BF16
    d = cfg.d
    # algorithmic work per step, by kernel
    flops_gemm = bytes_scan = 0.0
    n_loc = r1 - r0
    tmem_bytes = 0.0   # fp32 accumulators read out of TMEM by the main pass's epilogue
    for s, q in cells:
        ns = nsel[s]
        if cell_path[(s, q)] == vrs.PATH_GEMM:
            flops_gemm += 2.0 * q * ns * d
            # rows the main pass streams: the gathered selection iff it fits the
            # break-even buffer (vrs_api.cu), else every row (masked)
            cap = n_loc * 9 // 10 if q >= 1024 else (n_loc * 9 // 20 if q >= 256 else n_loc // 3)
            rows = ns if ns <= cap else n_loc
            tmem_bytes += 4.0 * 128 * ((q + 127) // 128) * rows
        else:
            bytes_scan += ns * (4.0 * d + 12) + q * 4.0 * d
    # the dominant kernel: the tensor-core main pass ("gemm.main", inside the "gemm" scope
    # that also holds the probe / threshold / gather launches), else the biggest scope
    # (any tensor-core cell: the main pass carries the step's algorithmic work -- on tiny
    # configs the probe or finalize may take longer, but they have no roofline of their own)
    flat = {kname: v for kname, v in prof.items() if kname != "gemm"}
    dominant = "gemm.main" if "gemm.main" in flat else (max(flat.items(), key=lambda kv: kv[1][0])[0] if flat else None)
    roof = None
    if dominant == "gemm.main":
        t_s = prof["gemm.main"][0] / 1e3 / nprof
        ach = flops_gemm / t_s / 1e12
        if ix.precision == vrs.PREC_BF16:   # kind::f16 on the bf16 shadow: the measured bf16 peak
            peak, peak_b, note, kind = (pk["bf16_tflops_sustained"], pk["bf16_tflops"],
                                        "measured bf16 (cuBLAS, MEASURED_PEAKS.json) sustained; burst beside", "bf16")
        else:
            peak, peak_b, note, kind = (tf32_peak_sus, tf32_peak_burst,
                                        "TF32 = measured bf16 sustained x nominal tf32/bf16 (1.1/2.25)", "TF32")
        roof = {"kernel": f"tc_topk_kernel main pass (tcgen05 {kind} + fused top-k)", "bound": "tensor",
                "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "traffic": None,
                "traffic_evidence": "profiles/r01_ncu_c2big_all_kernels.md: DRAM read / write of one C2 "
                                    "Q = 4096, s = 100 % main-pass launch (ncu --set full)",
                "peak_note": note, "frac_vs_burst_peak": ach / peak_b,
                "algorithmic": "2*Q*N_sel*d per cell, summed over the step's tensor-core cells, / main-pass time"}
    elif dominant is not None:
        t_s = prof[dominant][0] / 1e3 / nprof
        ach = bytes_scan / t_s / 1e9
        roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach / pk["hbm_gbs"], "traffic": None,
                "algorithmic": "N_sel*(4d+12) + 4*Q*d bytes per scan cell"}
    if roof is not None:
        roof["peak_source"] = pk["source"]
        if dominant == "gemm.main":
            # secondary ceiling of the fused epilogue: TMEM read-out, measured on this pool
            # at 310 B/clk/SM with the epilogue's 8 warps (tools/micro/tmem_bw.cu,
            # profiles/r01_s3_tmem_read_bw.txt) x 148 SMs x the max SM clock
            tpk = 310.0 * 148 * 1.965e9 / 1e12
            tach = tmem_bytes / (prof["gemm.main"][0] / 1e3 / nprof) / 1e12
            roof["secondary"] = {"bound": "tmem-read", "achieved": tach, "peak": tpk, "unit": "TB/s",
                                 "frac": tach / tpk,
                                 "note": "tcgen05.ld 32x32b.x32 alone, 8 warps/SM, measured (r01_s3_tmem_read_bw.txt)"}
        roof["kernel_share_of_step"] = {kname: v[0] / nprof / (ms / args.steps) for kname, v in prof.items()}

    # ---------------- per-cell timings (events around each cell)
    cell_out = []
    for c in cells:
        s, q = c
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run_cell(c)
        torch.cuda.synchronize()
        reps = 5
        a.record(stream)
        for _ in range(reps):
            run_cell(c)
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps / 1e3
        ns = nsel[s]
        fl = 2.0 * q * ns * d
        # algorithmic bytes: attribute columns, the selected rows once (bf16 shadow on the
        # bf16 tensor-core path, else fp32), the queries, the results
        esz = 2.0 if (vrs.last_path() == vrs.PATH_GEMM and ix.precision == vrs.PREC_BF16) else 4.0
        by = n_loc * sum(1 if cfg.attrs[i][0] == "u8" else 4 for i in range(len(cfg.attrs))) + ns * esz * d + q * 4.0 * d + q * k * 12
        cell_out.append({"sel": s, "q": q, "n_sel": ns, "ms": t * 1e3, "qps": q / t,
                         "path": "gemm" if vrs.last_path() == vrs.PATH_GEMM else "scan",
                         "hbm_frac": by / t / 1e9 / pk["hbm_gbs"], "tensor_frac": fl / t / 1e12 / tc_peak_sus})

    # ---------------- range (threshold) mode, SURVEY 8(f) NEXT #1 (not part of the step)
    range_out = []
    if world == 1 and cfg.metric != datagen.L2:
        s_all = cfg.sels[-1]
        q_r = min(256, max(cfg.qs))
        # the paper's threshold (cosine > 0.9) selects ~nothing on random
        # data; a second tau keeps tens of rows per query (C2 unit vectors: 0.35 ~ 4 sigma)
        for tau in (0.9, 0.35 if cfg.kind == "gauss_norm" else 0.9):
            ix.range_search(Qall[:q_r], preds[s_all], tau=tau, metric=metric)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 5
            for _ in range(reps):
                off, rid, rdist = ix.range_search(Qall[:q_r], preds[s_all], tau=tau, metric=metric)
            torch.cuda.synchronize()
            t = (time.perf_counter() - t0) / reps
            range_out.append({"tau": tau, "sel": s_all, "q": q_r, "ms": t * 1e3, "qps": q_r / t,
                              "results_per_query": rid.numel() / q_r,
                              "timing": "host wall clock (the call synchronises twice to size its output)"})
            if cfg.kind != "gauss_norm":
                break

    # ---------------- e2e through the public API with host buffers
    e2e = None
    h2d = sum(q * d * 4 for _, q in cells)
    d2h = sum(q * k * 12 for _, q in cells)
    Qh = Qall.cpu().pin_memory()
    # Pipelined like a serving loop: two sets of pinned result buffers; a step's
    # results are complete when its event fires, and the host waits on that event
    # only before it reuses the set (two steps later).
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
        if world > 1:   # one all-gather + merge for the step, results to the host
            mi, md = gather_merge(ids_all, dists_all, k, metric)
            q0 = 0
            for c in cells:
                hb[c][0].copy_(mi[q0:q0 + c[1]], non_blocking=True)
                hb[c][1].copy_(md[q0:q0 + c[1]], non_blocking=True)
                q0 += c[1]
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
           "pipelining": "2 pinned result sets, host waits on a step's event before reusing its set; "
                         "downloads overlap the next cell's kernels (host_async = 2, vrs_host_fence per step)",
           "d2h_bytes_per_step": d2h}

    # ---------------- sampled parity + CPU baseline (rank 0, N = 1)
    parity = None
    cpu = None
    if rank == 0 and world == 1 and not (args.no_parity and args.no_cpu_baseline):
        import oracle
        oracle.build()
        X_h, attrs_h = X.cpu().numpy(), [a.cpu().numpy() for a in attrs]
        Q_h = Qall[:64].cpu().numpy()
        if not args.no_parity:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from parity import check_topk
            checked = 0
            pcells = sorted({(cfg.sels[min(1, len(cfg.sels) - 1)], cfg.qs[min(1, len(cfg.qs) - 1)]),
                             (cfg.sels[-1], cfg.qs[-1])})
            for s, q in pcells:
                ids, dists = run_cell((s, q))
                torch.cuda.synchronize()
                nq = 3
                check_topk(ids[:nq].cpu().numpy(), dists[:nq].cpu().numpy(), X_h, attrs_h, preds[s], Q_h[:nq], k,
                           metric)
                checked += nq
            # A1 / A2 in full for every selectivity: bitmap words and count
            # bit-exact against the oracle's selection
            for s in cfg.sels:
                bm, cnt, _ = ix.select(preds[s])
                obm, ocnt, _ = oracle.select(attrs_h, n_loc, preds[s])
                gbm = bm.cpu().numpy().view(np.uint32)
                if int(cnt.item()) != ocnt or not np.array_equal(gbm, obm[: gbm.size]):
                    raise AssertionError(f"selection mismatch at s = {s}: count {int(cnt.item())} vs {ocnt}")
            parity = {"checked_queries": checked, "cells": [list(c) for c in pcells],
                      "bitmaps_checked": [float(x) for x in cfg.sels],
                      "rule": "SURVEY 8(c) c.5 (1e-3 rel dists, id sets within the k-th band); "
                              "bitmap + count bit-exact for every selectivity", "ok": True}
        if not args.no_cpu_baseline:
            threads = len(os.sched_getaffinity(0))
            v, t_all, desc, _ = oracle_sample(cfg, X_h, attrs_h, Q_h, 4, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                   "sample_seconds": t_all}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak" if cfg.shard_rows else "strong", "vs_baseline": None,
                "dtype": "bf16" if ix.precision == vrs.PREC_BF16 else "tf32",
                "dtype_note": "tensor-core selection operands (fp32 accumulate); returned dists re-scored in fp64 from fp32",
                "data": "synthetic", "config": workload_desc(cfg, world), "e2e": e2e,
                "gpu_launches": gpu_launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
                "timing": ("CUDA graph of the step (captured once, outside the timed region), replayed K times"
                           if graph is not None else "eager launches"),
                "parity": parity, "cells": cell_out, "range_search": range_out, "step_ms": [round(x, 4) for x in step_ms],
                "kernels_ms_per_step": {kname: v[0] / nprof for kname, v in prof.items()}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
