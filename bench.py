#!/usr/bin/env python3
"""bench.py — PiPNN index build on B200 (BASELINE.json metric: build points/s, leaf distance TFLOP/s,
% roofline, recall@10).

A step = one pipnn_build (all §8(a) rows: sketches, partition, leaf distance tiles + pick, HashPrune,
final prune, CSR) over one synthetic input resident in HBM. Default workload: BASELINE.json configs[4]
(C5: n=50M, d=128 uint8, L2, BIGANN-shaped 100k-cluster mixture, C_max 2048, l_max 96, R 32 — the largest
configuration that fits one GPU; configs[1..3] run with --config C2/C3/C4). Multi-GPU: one process per GPU
(torchrun), each rank builds its own independent replica of the workload (the build does not shard;
DESIGN.md "Multi-GPU"), value = all ranks' points / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

--impl reference times the CPU oracle (oracle/, the reference arm of this tier) on a bounded sample of the
same workload on the host cores; rank 0 only.
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

import synth  # noqa: E402

METRIC = "index build points/s and leaf distance TFLOP/s on 1 B200; % roofline; recall@10"
UNIT = "points/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload_desc(cfg: synth.Config) -> dict:
    return {"workload": f"{cfg.name}: n={cfg.n:,} d={cfg.d} {cfg.dtype} {cfg.metric}, {cfg.n_centres:,}-cluster "
                        f"synthetic mixture (BASELINE.json configs[{list(synth.CONFIGS).index(cfg.name.split('@')[0])}])",
            "n": cfg.n, "d": cfg.d, "dtype": cfg.dtype, "metric": cfg.metric, "c_max": cfg.c_max,
            "fanout": list(cfg.fanout), "k": cfg.k, "m": cfg.m, "l_max": cfg.l_max, "R": cfg.R,
            "alpha": f"{cfg.alpha_num}/{cfg.alpha_den}", "c_min": cfg.c_min, "leader_cap": cfg.leader_cap}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                if len(parts) >= 8:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def int8_peak_tops(dev) -> float:
    """Dense int8 tensor-core rate on this GPU, measured like MEASURED_PEAKS.json's bf16 figure (torch._int_mm
    8192^3, best of 10 after 3 warm-ups, CUDA events)."""
    import torch

    N = 8192
    a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device=dev).t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * N ** 3 / best / 1e9


def exact_knn(Xd, Qd, metric, k=10, qids=None, xchunk=1 << 21, qchunk=2048):
    """Exact k nearest of every query by a chunked fp32 GEMM over X (exact for uint8: every partial sum is an
    integer < 2^24); qids: the queries are these base points, themselves excluded. -> ids int64 [nq, k]."""
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    n, nq = Xd.shape[0], Qd.shape[0]
    out = torch.empty((nq, k), dtype=torch.int64, device=Xd.device)
    for q0 in range(0, nq, qchunk):
        Qf = Qd[q0:q0 + qchunk].float()
        q2 = (Qf * Qf).sum(1, keepdim=True)
        bd = torch.full((Qf.shape[0], k), float("inf"), device=Xd.device)
        bi = torch.full((Qf.shape[0], k), -1, dtype=torch.int64, device=Xd.device)
        for x0 in range(0, n, xchunk):
            Xf = Xd[x0:x0 + xchunk].float()
            D = -(Qf @ Xf.T) if metric == "mips" else q2 + (Xf * Xf).sum(1)[None] - 2 * (Qf @ Xf.T)
            if qids is not None:
                own = qids[q0:q0 + qchunk] - x0
                r = torch.nonzero((own >= 0) & (own < Xf.shape[0])).flatten()
                D[r, own[r]] = float("inf")
            d, i = torch.topk(D, k, dim=1, largest=False)
            cd, ci = torch.cat([bd, d], 1), torch.cat([bi, i + x0], 1)
            bd, sel = torch.topk(cd, k, dim=1, largest=False)
            bi = torch.gather(ci, 1, sel)
            del D, Xf
        out[q0:q0 + qchunk] = bi
    return out


def entry_point(Xd, metric, chunk=1 << 21) -> int:
    """The point nearest the dataset mean by (D, id) (R25; MIPS: argmax <x, mean>), fp64, chunked."""
    import torch

    n = Xd.shape[0]
    mean = torch.zeros(Xd.shape[1], dtype=torch.float64, device=Xd.device)
    for x0 in range(0, n, chunk):
        mean += Xd[x0:x0 + chunk].double().sum(0)
    mean /= n
    best, arg = None, 0
    for x0 in range(0, n, chunk):
        Xe = Xd[x0:x0 + chunk].double()
        v = -(Xe @ mean) if metric == "mips" else ((Xe - mean) ** 2).sum(1)
        j = int(torch.argmin(v).item())
        if best is None or float(v[j]) < best:
            best, arg = float(v[j]), x0 + j
    return arg


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_max(x: float, ws: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (torch.distributed all_reduce MAX; the identity at ws == 1)."""
    if ws <= 1:
        return float(x)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(ms_local: float, n_per_rank: int, ws: int, device=None):
    """Whole-job value of a weak-scaling step: every rank builds n_per_rank points; the job's step time is the
    slowest rank's (max over ranks), so value = n_per_rank * ws / max_ms."""
    ms_max = rank_max(ms_local, ws, device)
    return ms_max, n_per_rank * ws / (ms_max / 1e3)


def run_reference(args, cfg):
    """Reference arm: the CPU oracle, as it stands, on a bounded sample of the workload (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O

    n_s = args.ref_sample
    sub = cfg.scaled(n_s, n_centres=cfg.n_centres) if n_s < cfg.n else cfg  # the workload's first n_s points
    X = synth.gen_points(sub)
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.build(ds, sub.params())
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    val = sub.n / t
    cores = O.num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if cfg.dtype != "u8" else "int64", "data": "synthetic",
            "config": workload_desc(cfg),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"oracle build (partition, leaf pick, HashPrune, final prune) of the first "
                                       f"{sub.n:,} points of the {cfg.name} workload with the same parameters"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, n_sample, dev):
    """The oracle, as it stands, on the workload's first n_sample points (same parameters) on the host cores;
    the GPU builds the same sample and the two graphs are compared (identical CSR for uint8) and searched with
    the same queries and entry point (paired recall@10)."""
    import torch

    import oracle as O
    import paper_2602_21247_b200 as P

    sub = cfg.scaled(n_sample, n_centres=cfg.n_centres) if n_sample < cfg.n else cfg
    X = synth.gen_points(sub)
    ds = O.Dataset(X, metric=cfg.metric, mode="bf16")
    t0 = time.perf_counter()
    ref = O.build(ds, sub.params())
    dt = time.perf_counter() - t0
    base = {"value": sub.n / dt, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle", "cpu": cpu_model(),
            "sample": f"oracle build of the first {sub.n:,} points of the {cfg.name} workload, same parameters "
                      f"({dt:.1f} s)"}
    Xd = torch.from_numpy(X).to(dev)
    out = P.pipnn_build(Xd, P.build_params_from(sub.params()), metric=cfg.metric)
    rp, ci = out.row_ptr.cpu().numpy(), out.col_idx.cpu().numpy().view(np.uint32)
    same = bool(np.array_equal(rp, ref.row_ptr) and np.array_equal(ci, ref.col_idx))
    Qd = torch.from_numpy(synth.gen_queries(cfg, n_queries=1000)).to(dev)
    truth = exact_knn(Xd, Qd, cfg.metric)
    e = entry_point(Xd, cfg.metric)
    rows = {}
    rpo = torch.from_numpy(ref.row_ptr.astype(np.int64)).to(dev)
    cio = torch.from_numpy(ref.col_idx.view(np.int32)).to(dev)
    for L in (10, 32, 64, 128):
        a, _, _ = P.pipnn_search(Xd, out.row_ptr, out.col_idx, Qd, e, L, 10, cfg.metric)
        b, _, _ = P.pipnn_search(Xd, rpo, cio, Qd, e, L, 10, cfg.metric)
        ra = (a.long().unsqueeze(2) == truth.unsqueeze(1)).any(2).sum(1).double() / 10
        rb = (b.long().unsqueeze(2) == truth.unsqueeze(1)).any(2).sum(1).double() / 10
        d = ra - rb
        rows[str(L)] = {"gpu": round(float(ra.mean()), 4), "oracle": round(float(rb.mean()), 4),
                        "paired_diff": round(float(d.mean()), 5), "se": round(float(d.std() / len(d) ** 0.5), 5)}
    parity = {"n": sub.n, "csr_identical": same, "gpu_edges": int(rp[-1]), "oracle_edges": int(ref.row_ptr[-1]),
              "recall_at_10_paired": rows, "queries": 1000}
    return base, parity


def recall_eval(Xd, cfg, row_ptr, col_idx, n_queries, knn_queries=1_000_000):
    """recall@10 of the GPU graph over the L sweep (evaluation harness, not the method): queries from the
    config's generator, exact ground truth by a chunked fp32 torch GEMM over X (exact for uint8 data), entry
    point = the point nearest the dataset mean (R25), search by the library's batched beam search
    (pipnn_search, Alg. 1); plus the search's throughput (queries/s, CUDA events) at each L. Then the k-NN-graph
    task: base points queried on their own index, themselves excluded, over an L sweep up to the first
    L reaching recall@10 >= 0.95 (or 256, the kernel's limit): points/s on the first knn_queries base points and
    recall on 1,000 of them."""
    import torch

    import paper_2602_21247_b200 as P

    Q = synth.gen_queries(cfg, n_queries=n_queries)
    Qd = torch.from_numpy(Q).to(Xd.device)
    truth = exact_knn(Xd, Qd, cfg.metric)
    entry = entry_point(Xd, cfg.metric)
    recall, qps = {}, {}
    for L in (10, 32, 64, 128):
        P.pipnn_search(Xd, row_ptr, col_idx, Qd[:100], entry, L, 10, cfg.metric)  # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids, _, _ = P.pipnn_search(Xd, row_ptr, col_idx, Qd, entry, L, 10, cfg.metric)
        e1.record()
        torch.cuda.synchronize()
        qps[str(L)] = round(len(Q) / (e0.elapsed_time(e1) / 1e3))
        hit = (ids.long().unsqueeze(2) == truth.unsqueeze(1)).any(2).sum(1).float() / 10.0
        recall[str(L)] = round(float(hit.mean().item()), 4)
    nk = min(Xd.shape[0], knn_queries)
    g = torch.Generator(device="cpu").manual_seed(5)
    smp = torch.randperm(nk, generator=g)[:1000].to(Xd.device)
    gt = exact_knn(Xd, Xd[smp], cfg.metric, qids=smp)
    sweep = {}
    for L in (64, 128, 256):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gids, _, _ = P.pipnn_search(Xd, row_ptr, col_idx, Xd[:nk], entry, L, 10, cfg.metric, exclude_self=True)
        e1.record()
        torch.cuda.synchronize()
        rec = float(((gids[smp].long().unsqueeze(2) == gt.unsqueeze(1)).any(2).sum(1).float() / 10.0).mean())
        sweep[str(L)] = {"points_per_s": round(nk / (e0.elapsed_time(e1) / 1e3)), "recall_at_10_sample1000": round(rec, 4)}
        if rec >= 0.95:
            break
    first = next((int(L) for L, v in sweep.items() if v["recall_at_10_sample1000"] >= 0.95), None)
    return recall, qps, {"k": 10, "queried_points": nk, "L_sweep": sweep, "first_L_recall_ge_0.95": first}


def run_sharded(args, cfg):
    """--shard: ONE build of the workload sharded over the N ranks (paper_2602_21247_b200.sharded): rank 0
    partitions and broadcasts the LeafSet, each rank picks in its leaf range, one all_to_all routes the edges to the
    owners' ranks, each rank runs HashPrune + the final prune of its owners. value = n / max-over-ranks step time
    (strong scaling: the total work is fixed). e2e: each rank copies X in (pinned) and its CSR rows out."""
    import torch
    import torch.distributed as dist

    import paper_2602_21247_b200 as P
    from paper_2602_21247_b200 import sharded as SH

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % (29500 + os.getpid() % 1000), rank=0,
                                world_size=1)
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    X = synth.gen_points(cfg)  # every rank holds the same X (replicated, §8(e))
    Xh = torch.from_numpy(X).pin_memory()
    Xd = Xh.to(dev)
    params = P.build_params_from(cfg.params())

    def step():
        return SH.sharded_build(Xd, params, cfg.metric) if ws > 1 else SH.virtual_sharded_build(Xd, params, 1,
                                                                                                  cfg.metric)[0]
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = P.pipnn_launch_count()
    times = []
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = P.pipnn_launch_count() - launches0
    ms = statistics.mean(times)
    ms_max = rank_max(ms, ws, dev)
    rows_h = torch.empty(out.row_ptr.numel(), dtype=torch.int64).pin_memory()
    cols_h = torch.empty(max(1, out.col_idx.numel()), dtype=torch.int32).pin_memory()
    e2e = []
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        Xd.copy_(Xh, non_blocking=True)
        o = step()
        rows_h.copy_(o.row_ptr, non_blocking=True)
        cols_h[: o.col_idx.numel()].copy_(o.col_idx, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        e2e.append(e0.elapsed_time(e1))
    e2e_max = rank_max(statistics.mean(e2e), ws, dev)
    edges = torch.tensor([float(out.col_idx.numel())], device=dev)
    if ws > 1:
        dist.all_reduce(edges)
    if rank == 0:
        line = {"metric": METRIC, "value": cfg.n / (ms_max / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u8" if cfg.dtype == "u8" else "bf16", "data": "synthetic",
                "config": {**workload_desc(cfg), "parallelism": f"sharded x{ws}: leaf ranges + owner ranges, one "
                                                                f"all_to_all of edges (SURVEY 8(e))"},
                "e2e": {"value": cfg.n / (e2e_max / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(X.nbytes),
                        "d2h_bytes_per_step": int(rows_h.numel() * 8 + out.col_idx.numel() * 4),
                        "mode": "serial per rank: X H2D, sharded build, own CSR rows D2H"},
                "gpu_launches": int(launches), "graph_edges": int(edges.item()), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=100_000)
    ap.add_argument("--cpu-sample", type=int, default=1_000_000)
    ap.add_argument("--no-int8-peak", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--recall-queries", type=int, default=10000)
    ap.add_argument("--quant", action="store_true",
                    help="NEXT-2: float L2 leaves picked by per-leaf int8-quantised distances, re-ranked exactly")
    ap.add_argument("--shard", action="store_true",
                    help="one build sharded over the ranks (SURVEY §8(e), NEXT-4; strong scaling) instead of replicas")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.shard:
        run_sharded(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2602_21247_b200 as P

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)

    X = synth.gen_points(cfg, seed=rank)  # each rank: an independent replica of the workload
    Xh = torch.from_numpy(X).pin_memory()
    Xd = Xh.to(dev)
    pd = cfg.params()
    pd["quant"] = 1 if args.quant else 0
    params = P.build_params_from(pd)
    builder = P.Builder(Xd, params, metric=cfg.metric)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        out = builder(Xd)
    torch.cuda.synchronize()

    # ---------------- device-timed region (inputs resident in HBM)
    step_ms, stats = [], []
    launches0 = P.pipnn_launch_count()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = builder(Xd)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            stats.append(out.stats)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = P.pipnn_launch_count() - launches0
    ms = sum(step_ms) / len(step_ms)
    ms_max, value = job_throughput(ms, cfg.n, ws, dev)

    # ---------------- end-to-end through the public API with host buffers (pinned), copies inside
    n_rp = cfg.n + 1
    rp_h = torch.empty(n_rp, dtype=torch.int64).pin_memory()
    ci_h = torch.empty(cfg.n * cfg.R, dtype=torch.int32).pin_memory()
    e2e_ms, d2h = [], 0
    for _ in range(max(2, min(args.steps, 5))):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        Xd.copy_(Xh, non_blocking=True)
        o = builder(Xd)
        rp_h.copy_(o.row_ptr, non_blocking=True)
        ci_h[: o.n_edges].copy_(o.col_idx, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        d2h = n_rp * 8 + o.n_edges * 4
    _, e2e_serial = job_throughput(sum(e2e_ms) / len(e2e_ms), cfg.n, ws, dev)

    # ---------------- end-to-end, pipelined as a build service runs it: every step still copies its input
    # host->device and reads its CSR back, but on a copy stream, so the copy of step i+1's input and the read-back
    # of step i overlap build i (two device input buffers and two builders' outputs; skipped when memory is short).
    # (The library moves its own small uploads/read-backs with kernels, so they do not queue behind these copies
    # on the copy engines; splitting these copies into pieces did not help.)
    e2e_val, e2e_mode = e2e_serial, "serial: H2D, build, D2H per step on one stream"
    free_b, _ = torch.cuda.mem_get_info(dev)
    need = builder.ws_bytes + Xd.nbytes + builder.row_ptr.nbytes + builder.col_idx.nbytes
    fits = torch.tensor([1 if need < 0.8 * free_b else 0], device=dev)
    if ws > 1:
        dist.all_reduce(fits, op=dist.ReduceOp.MIN)  # every rank takes the same branch (collectives inside)
    if int(fits.item()):
        builder2 = P.Builder(Xd, params, metric=cfg.metric)
        Xd2 = torch.empty_like(Xd)
        bufs = [(Xd, builder), (Xd2, builder2)]
        cs = torch.cuda.Stream(dev)
        K = max(4, min(args.steps, 8))
        ev_h2d = [torch.cuda.Event() for _ in range(K)]
        ev_build = [torch.cuda.Event() for _ in range(K)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        builder2(Xd)  # warm the second builder
        flush.zero_()
        torch.cuda.synchronize()
        t0.record(cs)
        with torch.cuda.stream(cs):
            Xd.copy_(Xh, non_blocking=True)
            ev_h2d[0].record(cs)
        for i in range(K):
            xd, b = bufs[i % 2]
            if i + 1 < K:
                nx = bufs[(i + 1) % 2][0]
                with torch.cuda.stream(cs):
                    if i >= 1:
                        cs.wait_event(ev_build[i - 1])  # build i-1 is done with that input buffer
                    nx.copy_(Xh, non_blocking=True)
                    ev_h2d[i + 1].record(cs)
            stream.wait_event(ev_h2d[i])
            o = b(xd)  # returns when build i is complete
            ev_build[i].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_build[i])
                rp_h.copy_(o.row_ptr, non_blocking=True)
                ci_h[: o.n_edges].copy_(o.col_idx, non_blocking=True)
        t1.record(cs)
        torch.cuda.synchronize()
        _, e2e_val = job_throughput(t0.elapsed_time(t1) / K, cfg.n, ws, dev)
        e2e_mode = (f"pipelined over {K} steps: H2D of step i+1 and D2H of step i on a copy stream overlap build i "
                    "(first H2D and last D2H exposed)")
        del builder2, Xd2, bufs, b, xd  # (the builders' workspaces: the evaluation below needs the memory)

    if rank == 0:
        peaks, src = measured_peaks()
        st = stats[-1]
        tile_ms = statistics.mean(s["ms_leaf_tiles"] for s in stats)
        leaf_ops = 2.0 * st["leaf_pairs"] * cfg.d  # algorithmic: 2 s^2 d per leaf
        int8_meas = None
        if cfg.dtype == "u8":
            proxy = 2.0 * peaks["bf16_tflops"]  # nominal ratio 4.5/2.25 PF x measured bf16 burst
            if not args.no_int8_peak:
                try:
                    int8_meas = int8_peak_tops(dev)
                except Exception:
                    int8_meas = None
            # the larger of the measured int8 GEMM rate and the nominal-ratio proxy (the conservative peak)
            peak = max(proxy, int8_meas or 0.0)
            peak_note = (f"int8: max(measured torch._int_mm 8192^3 = {int8_meas and round(int8_meas, 1)} TOP/s, "
                         f"2 x bf16 burst {peaks['bf16_tflops']} ({src} MEASURED_PEAKS.json) = {proxy:.1f})")
        else:
            peak = peaks["bf16_tflops"]
            peak_note = f"bf16 burst ({src} MEASURED_PEAKS.json)"
        achieved = leaf_ops / (tile_ms / 1e3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "leaf_tile_traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    traffic = json.load(f).get(cfg.name)
            except Exception:
                traffic = None
        # per-pass HBM: algorithmic bytes / the stage's device time, against the measured copy
        # bandwidth. Occupied reservoir slots and degrees of the last build.
        bb = builder.debug_buffers(Xd, st)
        occ = int(bb["count"].long().sum().item())
        E = st["n_edges"]
        I = st["n_instances"]
        ebytes = 1 if cfg.dtype == "u8" else 2  # the path's row precision (bf16 for float data)
        row_b = cfg.d * ebytes
        kb = -(-cfg.d // 32) * 32 if cfg.dtype == "u8" else -(-cfg.d // 16) * 32 + 32
        ne = out.n_edges
        stg = {k: statistics.mean(s[k] for s in stats) for k in ("ms_prep", "ms_partition", "ms_leaf",
                                                               "ms_leaf_tiles", "ms_hashprune", "ms_final",
                                                               "ms_total")}
        hbm = peaks["hbm_gbs"]

        def pas(nbytes, ms, what):
            gbs = nbytes / (ms / 1e3) / 1e9 if ms > 0 else None
            return {"algorithmic_bytes": int(nbytes), "ms": round(ms, 4), "achieved_gbs": gbs and round(gbs, 1),
                    "peak_gbs": hbm, "frac": gbs and round(gbs / hbm, 4), "bytes": what}

        hbm_passes = {
            "leaf_gather": pas(I * (row_b + kb), stg["ms_leaf"] - stg["ms_leaf_tiles"],
                               "X rows gathered (d x elem) + tiled rows written (Kb) per instance"),
            "hashprune": pas(16 * E + 8 * occ + 4 * cfg.n, stg["ms_hashprune"],
                             "8-B edge key written by the emit and read by the merge per streamed edge + 8 B per "
                             "occupied slot written + count"),
            "final_prune": pas(occ * (row_b + 8) + ne * 4 * 3 + cfg.n * 16, stg["ms_final"],
                               "candidate rows gathered + reservoir slots read per occupied slot; admitted ids "
                               "written, re-read and copied into the CSR; degree + row_ptr per point"),
        }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8" if cfg.dtype == "u8" else "bf16", "data": "synthetic",
            "config": {**workload_desc(cfg), "parallelism": f"replicas x{ws} (independent builds)",
                       "l2": "flushed between timed steps (512 MB write)",
                       "leaf_pick": "int8-quantised + exact re-rank (NEXT-2)" if args.quant else "exact"},
            "roofline": {"bound": "tensor",
                         "kernel": ("dist_topk_uf2_kernel<8> (folded uint8 leaf tiles + fused pick, four epilogue "
                                    "warpgroups)" if cfg.dtype == "u8" and cfg.metric == "l2" and cfg.k <= 8
                                    and not args.quant else "dist_topk_kernel (leaf distance tiles + fused pick)"),
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s" if cfg.dtype != "u8" else "TOP/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_note,
                         "algorithmic_ops_per_launch": leaf_ops, "ms_per_launch": tile_ms,
                         "int8_measured_tops": int8_meas},
            "hbm_passes": hbm_passes,
            "stages_ms": {k: round(v, 4) for k, v in stg.items()},
            "counts": {**{k: st[k] for k in ("n_leaves", "n_instances", "n_edges", "max_leaf", "depth")},
                       "occupied_slots": occ, "graph_edges": int(ne)},
            "leaf_tflops": achieved,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": int(d2h),
                    "mode": e2e_mode, "serial_value": e2e_serial},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        # the evaluation needs memory: keep the graph, release the builder's workspace
        g_rp, g_ci = out.row_ptr.clone(), out.col_idx.clone()
        del out, bb, builder
        torch.cuda.empty_cache()
        if args.recall_queries > 0:
            try:
                rec, qps, knn = recall_eval(Xd, cfg, g_rp, g_ci, args.recall_queries)
                line["recall_at_10"] = rec
                line["search_qps"] = qps
                line["knn_graph_task"] = knn
                line["recall_queries"] = args.recall_queries
            except Exception as ex:  # evaluation is reported, never gates the timing
                line["recall_at_10"] = f"failed: {ex}"
        if not args.no_cpu_baseline:
            try:
                del g_rp, g_ci
                torch.cuda.empty_cache()
                line["cpu_baseline"], line["sample_parity"] = cpu_baseline(cfg, args.cpu_sample, dev)
            except Exception as ex:
                line["cpu_baseline"] = f"failed: {ex}"
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
