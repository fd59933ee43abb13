#!/usr/bin/env python
"""Benchmark of the Sinnamon hot path on B200 (contract: one JSON line on rank 0).

Default workload (BASELINE.json configs[4], "c5" — the largest single-GPU config by bytes and the
north star's HBM gate): 4M documents, n = 100,000, doc nnz ~ Poisson(250) with
Zipf(0.8) coordinates, Laplace(0,1) values; m = 256, h = 3; 1,024-query batches with nnz ~
Poisson(100); k = 100, k' = 2,000, exact re-rank.  The same line carries config 3 (configs[2], the
largest by documents, bound by Alg. 6's update rate) under "also" (--also c3; --also none skips it).
A step = one search batch of 1,024 queries through the whole path (S0 prep, S1 postings walk +
decode + accumulate, S2 top-k', S3 re-rank, S4 top-k); the index (built before timing, 100K-document
insert batches, timed separately as insert docs/s) and the query batches are resident in HBM when the
timed region starts.  The index (> 15 GB) exceeds the 126 MB L2, so no flush is needed between steps.

  --config tiny|c2|c3|c5   the BASELINE.json configs (same JSON line; evidence in profiles/)
  --config c4              the streaming protocol: rounds of insert 100K -> delete 1% of live ->
                           search 1,024 queries, 0 -> 4M documents; value = queries / search time
                           over all rounds, with the per-round curve (insert docs/s, QPS vs size)

  --impl sinn       (default) the CUDA path through the C ABI
  --impl reference  the CPU oracle (oracle/) on the host cores, as it stands: the tier's
                    reference arm (rank 0 only; other ranks exit 0)
  --shard           document shards instead of replicas (one candidate all-gather per batch, §8(e))
Multi-GPU: every rank holds a full replica of the index and searches its own query batches
(independent problems, no data-path collective): value = all queries / max-rank time.  Launched with
torchrun, or `--gpus N` alone (WORLD_SIZE unset): bench.py then starts the N ranks itself through
torch.distributed.run on 127.0.0.1.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# load every kernel of libsinn.so when the context is created rather than at its first launch
# (CUDA's lazy module loading would otherwise put a kernel's first load inside a timed insert batch)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "queries/sec (batch 1024) + recall@10 vs exact; scoring HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["sinn", "reference"], default="sinn")
    ap.add_argument("--config", default="c5")
    ap.add_argument("--also", default=None, help="extra config measured in the same run and reported under "
                                                 "'also' (default c3 with --config c5; 'none' to skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--docs", type=int, default=None, help="override the config's document count (profiling only)")
    ap.add_argument("--recall-queries", type=int, default=None)
    ap.add_argument("--cpu-sample-queries", type=int, default=512)
    ap.add_argument("--cpu-sample-docs", type=int, default=None,
                    help="the oracle baseline's index: the first D documents of the workload when the config "
                         "holds more (its per-query work is proportional to the index size; QPS is scaled by D/N); "
                         "default: as many documents as hold 120 M entries (the full index of configs 1 and 2)")
    ap.add_argument("--ref-step-queries", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--bf16", action="store_true",
                    help="bfloat16 sketch cells with directed rounding (SINN_SKETCH_BF16, F3 / DESIGN.md R21); "
                         "BASELINE.json's configs are fp32, so this is an extra line, not the default")
    ap.add_argument("--graph", action="store_true",
                    help="replay each timed search batch from a CUDA graph captured around the SINN_SEARCH_NOSYNC call "
                         "(one graph per resident batch; the launch-bound config 1 is where it pays); an extra line")
    ap.add_argument("--shard", action="store_true",
                    help="document sharding (SURVEY §8(e), DESIGN.md §9): the config's documents are split over the "
                         "ranks by id %% W and every rank scores the SAME query batches; per-shard top-k' lists are "
                         "all-gathered, merged, re-ranked by their owners, and the top-k lists merged (strong "
                         "scaling; an extra line, the default stays replicas)")
    ap.add_argument("--containers", action="store_true",
                    help="bitmap containers for dense tile lists (SINN_BITMAP_CONTAINERS, F3 / DESIGN.md §5.7)")
    return ap.parse_args()


_DESC = {
    "tiny": "BASELINE.json configs[0] (Tiny) — {N:,} docs, n={n:,}, doc nnz~U{{20..60}} uniform coords, N(0,1) fp32; "
            "m={m}, h={h}; {batch} queries nnz=10",
    "c2": "BASELINE.json configs[1] — {N:,} docs, n={n:,}, doc nnz~Poisson(120) uniform coords, N(0,1) fp32; "
          "m={m}, h={h}; batch {batch} queries nnz~Poisson(40)",
    "c3": "BASELINE.json configs[2] — {N:,} docs, n={n:,}, doc nnz~LogNormal(mean 120, sigma 0.5) clipped [5,600], "
          "Zipf(1.1) coords, LogNormal(0,1) fp32; Sinnamon+ (upper only), m={m}, h={h}; batch {batch} queries "
          "nnz~Poisson(43) same Zipf",
    "c4": "BASELINE.json configs[3] (streaming) — config-2 law grown 0 -> {N:,} docs in 100,000-doc inserts, delete "
          "1% of live + search {batch} queries after each insert; m={m}, h={h}",
    "c5": "BASELINE.json configs[4] — {N:,} docs, n={n:,}, doc nnz~Poisson(250) Zipf(0.8) coords, Laplace(0,1) fp32; "
          "m={m}, h={h}; batch {batch} queries nnz~Poisson(100) same Zipf",
}


def workload_desc(cfg, bf16=False) -> str:
    body = _DESC.get(cfg.name, cfg.name).format(N=cfg.N, n=cfg.n, m=cfg.m, h=cfg.h, batch=cfg.batch)
    cells = "; bfloat16 sketch cells (SINN_SKETCH_BF16, directed rounding)" if bf16 else ""
    return f"{cfg.name}: {body}; k={cfg.k}, k'={cfg.kprime}, exact re-rank{cells}"


def l2_note(cfg) -> str:
    """The timing rule's L2 statement, from the index's size (sketch columns + ~12 B per stored entry)."""
    nnz = {"tiny": 40, "c2": 120, "c3": 120, "c4": 120, "c5": 250}.get(cfg.name, 120)
    gb = cfg.N * (cfg.m * (1 if cfg.upper_only else 2) * 4 + nnz * 12) / 1e9
    if gb > 0.5:
        return f"inputs larger than L2 (index ~{gb:.1f} GB against 126 MB); no flush"
    return (f"index ~{gb * 1e3:.0f} MB fits the 126 MB L2: steps run L2-warm, no flush (this config is launch-latency-bound, "
            f"not bandwidth-bound; its roofline fraction is reported for completeness only)")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def sm_clock_mhz():
    """Max SM clock for the FP32 update roof: MEASURED_PEAKS.json sm_max_mhz, else the device's."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("sm_max_mhz"):
            return float(d["sm_max_mhz"]), "MEASURED_PEAKS.json sm_max_mhz"
    import torch
    return torch.cuda.get_device_properties(0).clock_rate / 1e3, "cudaDeviceProp clockRate"


def insert_alg_bytes(cfg, nnz_total, docs):
    """Insert's algorithmic bytes (SURVEY §8(d) "Insert"): per entry 8 B read (index + value), 4 B
    postings write, 8 B raw-store write; per document 4 m sides B of sketch column and 4 B of id."""
    sides = 1 if cfg.upper_only else 2
    return nnz_total * (8 + 4 + 8) + docs * (4.0 * cfg.m * sides + 4)


class ClockSampler:
    """nvidia-smi samples during the timed region (clocks, power, throttle reasons)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.15)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(cfg, term_len, qp, qi, qv, mean_doc_nnz, cell_bytes=4):
    """Per-batch algorithmic bytes:
    ids 4 B per posting of every distinct batch term; sketch cells 4 B x h per posting per needed
    sign side, capped by streaming the needed halves of the whole sketch once; re-rank
    B k' (8 psi_d + 8)."""
    nz = qv != 0
    j, v = qi[nz], qv[nz]
    pos = np.zeros(cfg.n, bool)
    neg = np.zeros(cfg.n, bool)
    pos[j[v > 0]] = True
    if not cfg.upper_only:
        neg[j[v < 0]] = True
    terms = pos | neg
    L = term_len.astype(np.float64)
    b_ids = 4.0 * L[terms].sum()
    gather = float(cell_bytes) * cfg.h * (L[pos].sum() + L[neg].sum())
    stream = float(cell_bytes) * cfg.m * cfg.N * (int(pos.any()) + int(neg.any()))
    b_sk = min(gather, stream)
    nq = qp.size - 1
    b_rr = nq * cfg.kprime * (8.0 * mean_doc_nnz + 8.0)
    # Alg. 6's (document, query) updates: every posting of a batch term times the batch queries
    # holding it (per needed sign; SURVEY §8(d) "Updates")
    qf_pos = np.bincount(j[v > 0], minlength=cfg.n).astype(np.float64)
    qf_neg = np.zeros(cfg.n) if cfg.upper_only else np.bincount(j[v < 0], minlength=cfg.n).astype(np.float64)
    upd = float((L * (qf_pos + qf_neg)).sum())
    return {"ids": b_ids, "sketch": b_sk, "rerank": b_rr, "updates": upd}



def library_warmup(cfg, table, dev, bf16):
    """Warm-up outside every timed region, called after the index's capacity reservation: a
    throwaway index of the same shape takes one insert batch and a delete, so first-use costs (the
    stream-ordered pool mapping memory for the insert workspace, first launches) are not charged to
    the first timed insert; the memory it frees stays in the pool for the real index."""
    import torch
    import paper_2301_10622_b200 as sinn
    W = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=bf16)
    wc = min(cfg.insert_batch, cfg.N)
    wp, wx, wv = datagen.docs(cfg, 0, wc)
    W.insert(torch.from_numpy(wp).to(dev), torch.from_numpy(wx).to(dev), torch.from_numpy(wv).to(dev),
             torch.arange(0, wc, dtype=torch.int32, device=dev))
    W.delete(torch.arange(0, min(wc, 1000), dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    W.close()
    torch.cuda.synchronize()

def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---- replicas: every rank holds the whole index and searches its own query batches;
# the only collectives are the timing barrier and the max over ranks (no data-path exchange)
def query_batch_start(rank: int, nb: int, b: int, batch: int) -> int:
    """First query row (in the config's seeded query stream) of rank `rank`'s b-th batch: the
    ranks' batches are disjoint, so the job's throughput counts every rank's queries."""
    return (rank * nb + b) * batch


def max_over_ranks(value: float, ws: int, device=None) -> float:
    """The job's time is the slowest rank's (max all-reduce); identity at ws == 1."""
    if ws <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_qps(batch: int, steps: int, ws: int, max_ms: float) -> float:
    """Whole-job throughput: all ranks' queries over the slowest rank's time."""
    return batch * steps * ws / (max_ms / 1e3)


# ------------------------------------------------------------------------------------------ oracle sample
def cpu_sample_docs(args, cfg) -> int:
    """--cpu-sample-docs, or the documents that hold ~120 M entries (~30 s of oracle inserts)."""
    if args.cpu_sample_docs:
        return args.cpu_sample_docs
    mean_nnz = float(np.diff(datagen.docs(cfg, 0, min(cfg.N, 5_000))[0]).mean())
    return int(min(cfg.N, max(100_000, 120e6 / max(mean_nnz, 1.0))))


def oracle_sample_index(cfg, table, max_docs, bf16=False):
    """The oracle (as it stands) over the first min(N, max_docs) documents of the workload; returns
    (index, documents held, insert seconds).  Its per-query work (Alg. 6 walks every posting of the
    query's terms; Alg. 3 scans every document) is proportional to the documents it holds, so a
    sub-index's QPS times D/N estimates the full index's — the bounded sample the contract allows."""
    import oracle
    D = min(cfg.N, max_docs)
    O = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=bf16)
    t_ins = 0.0
    for s0 in range(0, D, cfg.insert_batch):
        c = min(cfg.insert_batch, D - s0)
        ip, ix, v = datagen.docs(cfg, s0, c)
        t0 = time.perf_counter()
        assert O.insert(ip, ix, v, np.arange(s0, s0 + c, dtype=np.uint32)) == oracle.OK
        t_ins += time.perf_counter() - t0
    return O, D, t_ins


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    import oracle
    cfg = datagen.CONFIGS[args.config]
    table = datagen.hash_table(cfg)
    O, D, _ = oracle_sample_index(cfg, table, cpu_sample_docs(args, cfg), args.bf16)
    scale = D / cfg.N
    nqs = args.ref_step_queries
    cores = oracle.default_threads()
    # bound the run: a probe of `cores` queries sizes the step so that warm-up + timed steps stay
    # within ~150 s whatever --steps asks for (each step is a bounded sample of the workload)
    pp, pi_, pv = datagen.queries(cfg, 0, cores)
    t0 = time.perf_counter()
    O.search(pp, pi_, pv, cfg.k, cfg.kprime, cfg.rerank, cores)
    per_q = (time.perf_counter() - t0) / cores
    nqs = int(max(1, min(nqs, 150.0 / max(per_q, 1e-9) / (args.steps + args.warmup))))
    qp, qi, qv = datagen.queries(cfg, 0, nqs * (args.steps + args.warmup))

    def step(t):
        a, b = qp[t * nqs], qp[(t + 1) * nqs]
        O.search(qp[t * nqs:(t + 1) * nqs + 1] - a, qi[a:b], qv[a:b], cfg.k, cfg.kprime, cfg.rerank, cores)

    for t in range(args.warmup):
        step(t)
    t0 = time.perf_counter()
    for t in range(args.warmup, args.warmup + args.steps):
        step(t)
    el = time.perf_counter() - t0
    qps = nqs * args.steps / el * scale
    sample = (f"{nqs} queries of the {cfg.name} workload per step over the first {D:,} of its {cfg.N:,} documents; "
              f"QPS x {scale:g} (per-query work is proportional to the documents held)" if D < cfg.N else
              f"{nqs} queries of the {cfg.name} workload per step over the full {cfg.N:,}-doc index")
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps / scale,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            # the CUDA arm's config (the workload this line stands for); each step is a bounded sample of it
            "config": {"workload": workload_desc(cfg, args.bf16), "batch": cfg.batch, "k": cfg.k, "kprime": cfg.kprime,
                       "rerank": cfg.rerank, "l2": l2_note(cfg),
                       "parallelism": f"replicas x{ws}, query batches sharded across ranks"},
            "step_sample_queries": nqs,
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ CUDA arm
def run_sinn(args):
    import torch
    import torch.distributed as dist

    import paper_2301_10622_b200 as sinn

    ws, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    cfg = datagen.CONFIGS[args.config]
    if args.docs:
        import dataclasses
        cfg = dataclasses.replace(cfg, N=args.docs)
    if cfg.name == "c4":
        table = datagen.hash_table(cfg)
        G = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=args.bf16)
        rc = run_streaming(args, cfg, table, dev, stream, G, ws, rank)
        if ws > 1:
            dist.destroy_process_group()
        return rc
    if args.shard:
        rc = run_sharded(args, cfg, ws, rank, local, dev, stream)
        if ws > 1:
            dist.destroy_process_group()
        return rc
    line = measure(args, cfg, ws, rank, local, dev, stream, cpu=True)
    if args.also is None:  # config 3 rides along with the default config only
        args.also = "c3" if cfg.name == "c5" else "none"
    also = [c for c in (args.also or "").split(",") if c and c != "none" and c != cfg.name]
    if also and not args.docs:
        line["also"] = {}
        for name in also:
            sub = measure(args, datagen.CONFIGS[name], ws, rank, local, dev, stream, cpu=False)
            keep = ("value", "unit", "ms_per_step", "config", f"recall@{datagen.CONFIGS[name].k}", "recall", "insert",
                    "roofline", "roofline_update", "roofline_step", "kernels", "e2e", "gpu_launches", "clocks")
            line["also"][name] = {k_: sub.get(k_) for k_ in keep}
            line["gpu_launches_also"] = sub.get("gpu_launches")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def measure(args, cfg, ws, rank, local, dev, stream, cpu=True):
    """Build cfg's index on this rank's GPU, time args.steps search batches, and return the JSON line."""
    import torch
    import torch.distributed as dist

    import paper_2301_10622_b200 as sinn

    table = datagen.hash_table(cfg)
    G = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=args.bf16, containers=args.containers)

    # ---- build the index (insert batches of 100K docs); inputs uploaded first, insert timed on the device
    term_len = np.zeros(cfg.n, np.int64)
    # bulk load: capacity for the whole index up front (expected entries x 1.05)
    mean_nnz = float(np.diff(datagen.docs(cfg, 0, min(cfg.N, 20_000))[0]).mean())
    G.reserve(cfg.N, int(cfg.N * mean_nnz * 1.05))
    torch.cuda.synchronize()
    library_warmup(cfg, table, dev, args.bf16)
    ins_ms = 0.0
    ins_batches_ms = []
    nnz_total = 0
    gc.collect()
    gc.disable()  # no collector pause inside a timed insert (host stalls land in the event interval)
    G.profile(True)
    for s in range(0, cfg.N, cfg.insert_batch):
        c = min(cfg.insert_batch, cfg.N - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        term_len += np.bincount(ix, minlength=cfg.n)
        nnz_total += ix.size
        t = (torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), torch.from_numpy(v).to(dev),
             torch.arange(s, s + c, dtype=torch.int32, device=dev))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        G.insert(*t)
        e1.record(stream)
        torch.cuda.synchronize()
        ins_ms += e0.elapsed_time(e1)
        ins_batches_ms.append(round(e0.elapsed_time(e1), 3))
    ins_prof = G.profile_read()
    G.profile(False)
    gc.enable()
    insert_dps = cfg.N / (ins_ms / 1e3)
    mean_doc_nnz = nnz_total / cfg.N
    peak, peak_src = peaks()
    ins_bytes = insert_alg_bytes(cfg, nnz_total, cfg.N)
    ins_roof = {"bound": "hbm", "achieved": ins_bytes / (ins_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                "alg_bytes_per_doc": ins_bytes / cfg.N, "peak_source": peak_src,
                "note": "whole insert call (validation round trip included) over the algorithmic bytes of "
                        "SURVEY §8(d): 20 B per entry + 4 m sides + 4 B per document"}
    ins_roof["frac"] = ins_roof["achieved"] / peak

    # ---- query batches (distinct per rank and per step), resident on the device
    nb = min(args.steps + args.warmup, 16)
    batches = []
    for b in range(nb):
        qp, qi, qv = datagen.queries(cfg, query_batch_start(rank, nb, b, cfg.batch), cfg.batch)
        batches.append(((qp, qi, qv), (torch.from_numpy(qp).to(dev), torch.from_numpy(qi).to(dev),
                                       torch.from_numpy(qv).to(dev))))
    out = (torch.empty((cfg.batch, cfg.k), dtype=torch.int32, device=dev),
           torch.empty((cfg.batch, cfg.k), dtype=torch.float32, device=dev))
    alg = [algorithmic_bytes(cfg, term_len, *batches[b][0], mean_doc_nnz, 2 if args.bf16 else 4) for b in range(nb)]

    def step(t):
        G.search(*batches[t % nb][1], cfg.k, cfg.kprime, cfg.rerank, out=out, sync=False)

    graphs = None
    if args.graph:
        # the NOSYNC search has no host round trip and, once warmed, no allocation: capture one graph per
        # resident batch on this stream and replay it (profile events are not recorded inside a graph, so
        # the per-phase numbers of this line are absent and the roofline uses the whole step)
        side = torch.cuda.Stream()  # (capture needs a non-default stream; the replays run on `stream`)
        side.wait_stream(stream)
        graphs = []
        with torch.cuda.stream(side):
            for t in range(nb):
                step(t)
            G.sync()
            torch.cuda.synchronize()
            for t in range(nb):
                g_ = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_, stream=side):
                    step(t)
                graphs.append(g_)
        stream.wait_stream(side)
        torch.cuda.synchronize()
        direct_step = step

        def step(t):  # noqa: F811
            graphs[t % nb].replay()

    for t in range(args.warmup):
        step(t)
    G.sync()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    gc.collect()
    gc.disable()
    G.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(args.steps):
        step(args.warmup + t)
    e1.record(stream)
    torch.cuda.synchronize()
    G.sync()
    gc.enable()
    el_ms = e0.elapsed_time(e1)
    prof = G.profile_read()
    G.profile(False)
    clk = clocks.stop()
    if graphs is not None:
        # a replayed graph records no phase events: the per-phase times and launch counts of this line come
        # from the same steps issued directly right after the timed region (the timed value is the replay's)
        G.profile(True)
        for t in range(args.steps):
            direct_step(args.warmup + t)
        G.sync()
        prof = G.profile_read()
        G.profile(False)
    el_ms = max_over_ranks(el_ms, ws, dev)
    if ws > 1:
        dist.barrier()
    qps = job_qps(cfg.batch, args.steps, ws, el_ms)

    # ---- end to end through the C ABI with HOST buffers (H2D of queries + D2H of results inside)
    hout = (np.empty((cfg.batch, cfg.k), np.uint32), np.empty((cfg.batch, cfg.k), np.float32))
    for t in range(2):
        G.search_host(*batches[t % nb][0], cfg.k, cfg.kprime, cfg.rerank, out=hout)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for t in range(args.e2e_steps):
        G.search_host(*batches[t % nb][0], cfg.k, cfg.kprime, cfg.rerank, out=hout)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    e2e_ms = max_over_ranks(e2e_ms, ws, dev)
    e2e_qps = job_qps(cfg.batch, args.e2e_steps, ws, e2e_ms)
    qp0, qi0, qv0 = batches[0][0]
    h2d = qp0.nbytes + qi0.nbytes + qv0.nbytes
    d2h = cfg.batch * cfg.k * 8

    # ---- roofline of the dominant search phase (CUDA events around each phase, timed region)
    search_phases = ("prep", "init", "score", "select", "rerank", "final")
    dom = "score"  # the S1+S2 pass: the kernel the roofline is reported for (dominant at every config but tiny)
    a_tot = {k_: float(np.mean([a[k_] for a in alg])) for k_ in ("ids", "sketch", "rerank")}  # bytes
    per_step_alg = {"prep": 0.0, "init": 0.0, "score": a_tot["ids"] + a_tot["sketch"], "select": 0.0,
                    "rerank": a_tot["rerank"], "final": 0.0}
    ms, calls, _ = prof[dom]
    # with head terms the threshold's large sample keeps its documents' score rows and the full pass skips
    # the sampled tiles (every stride-th): the score phase then reads (1 - 1/stride) of the ids and cells
    st_ = G.stats()
    covered = 1.0 - 1.0 / st_["sample_stride"] if st_["sample_rows_kept"] and st_["sample_stride"] > 1 else 1.0
    per_step_alg["score"] *= covered
    per_launch_bytes = per_step_alg[dom] * args.steps / max(calls, 1)
    achieved = per_launch_bytes / (ms / max(calls, 1) / 1e3) / 1e9 if ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):  # dram__bytes_read.sum + dram__bytes_write.sum per launch, from an ncu --set full capture
        traffic = json.load(open(tpath)).get(cfg.name + ("_bf16" if args.bf16 else ""), {}).get(dom, {}).get("bytes_per_launch")
    kname = sinn_score_kernel_name(cfg)
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": per_launch_bytes, "tiles_covered_by_this_pass": covered}
    # the update roofline (configs 3 and 5 are bound by updates, not HBM): Alg. 6's
    # (document, query) updates per score pass / its time, against one FFMA per update at the FP32
    # peak (SMs x 128 lanes x the max SM clock) — the "alu" bound for this pass
    upd_step = float(np.mean([a["updates"] for a in alg])) * covered
    upd_launch = upd_step * args.steps / max(calls, 1)
    mhz, mhz_src = sm_clock_mhz()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    ffma_peak = nsm * 128 * mhz * 1e6
    roof_upd = {"bound": "alu", "kernel": kname, "updates_per_launch": upd_launch,
                "achieved": upd_launch / (ms / max(calls, 1) / 1e3) if ms > 0 else 0.0,
                "peak": ffma_peak, "unit": "updates/s",
                "peak_source": f"{nsm} SMs x 128 FP32 lanes x {mhz:.0f} MHz ({mhz_src}), one FFMA per update"}
    roof_upd["frac"] = roof_upd["achieved"] / ffma_peak
    step_alg = sum(a_tot.values())
    roof_step = {"alg_bytes_per_step": step_alg, "achieved": step_alg / (el_ms / args.steps / 1e3) / 1e9,
                 "unit": "GB/s", "peak": peak}
    roof_step["frac"] = roof_step["achieved"] / peak
    kernels = {p: {"ms_per_step": prof[p][0] / args.steps, "launches_per_step": prof[p][2] / args.steps}
               for p in search_phases}
    gpu_launches = int(sum(prof[p][2] for p in search_phases))

    # ---- recall@k of a whole batch against the GPU's exact MIPS (sinn_search_exact, LinScan on the
    # same walk; parity-tested against the oracle's exact search), outside the timed region
    qb = batches[0][1]
    ai, _ = G.search(*qb, cfg.k, cfg.kprime, cfg.rerank)
    xi, _ = G.search_exact(*qb, cfg.k)
    ai, xi = ai.cpu().numpy(), xi.cpu().numpy()
    nq_rec = ai.shape[0]
    recall_gpu = float(np.mean([len(set(ai[q].tolist()) & set(xi[q].tolist())) / cfg.k for q in range(nq_rec)]))

    # ---- the CPU oracle baseline (rank 0, N = 1) on a bounded sample: the oracle over the first
    # --cpu-sample-docs documents (the full index when it holds fewer), QPS scaled by D/N; recall@k vs
    # the oracle's exact search on a query sample when the oracle holds the full index
    recall = None
    cpu_line = None
    if cpu and rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        cores = oracle.default_threads()
        O, D, t_ins = oracle_sample_index(cfg, table, cpu_sample_docs(args, cfg), args.bf16)
        qp, qi, qv = batches[0][0]
        R = None
        if D == cfg.N:
            R = min(args.recall_queries or 32, cfg.batch)
            sub = slice(0, R + 1)
            eids, _ = O.exact(qp[sub], qi[:qp[R]], qv[:qp[R]], cfg.k, cores)
            gi, _ = G.search_host(qp[sub], qi[:qp[R]], qv[:qp[R]], cfg.k, cfg.kprime, cfg.rerank)
            recall = float(np.mean([len(set(gi[q].tolist()) & set(eids[q].tolist())) / cfg.k for q in range(R)]))
        S = min(args.cpu_sample_queries if D == cfg.N else 64, cfg.batch)
        t0 = time.perf_counter()
        O.search(qp[:S + 1], qi[:qp[S]], qv[:qp[S]], cfg.k, cfg.kprime, cfg.rerank, cores)
        cpu_s = time.perf_counter() - t0
        scale = D / cfg.N
        sample = (f"{S} queries of batch 0 over the full {cfg.N:,}-doc index (fp64 Alg. 6+7, all cores)" if D == cfg.N else
                  f"{S} queries of batch 0 over the first {D:,} of the {cfg.N:,} documents (fp64 Alg. 6+7, all cores); "
                  f"QPS x {scale:g}: the oracle's per-query work is proportional to the documents it holds")
        cpu_line = {"value": S / cpu_s * scale, "unit": "queries/s", "cores": cores, "kind": "oracle",
                    "sample": sample, "insert_docs_per_s": D / t_ins, "recall_sample_queries": R}
        del O

    line = {"metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg, args.bf16), "batch": cfg.batch, "k": cfg.k, "kprime": cfg.kprime,
                       "rerank": cfg.rerank, "l2": l2_note(cfg),
                       "parallelism": f"replicas x{ws}, query batches sharded across ranks"},
            f"recall@{cfg.k}": recall if recall is not None else recall_gpu,
            "recall": {"vs_oracle_exact": recall, "oracle_sample_queries": cpu_line and cpu_line.get("recall_sample_queries"),
                       "vs_gpu_exact": recall_gpu, "gpu_exact_queries": int(nq_rec)},
            "insert": {"value": insert_dps, "unit": "docs/s", "batch": cfg.insert_batch, "roofline": ins_roof,
                       "phases_ms": {p: ins_prof[p][0] for p in ("validate", "sketch", "postings", "raw")},
                       "batches_ms": ins_batches_ms},
            "roofline": roof, "roofline_step": roof_step, "roofline_update": roof_upd, "kernels": kernels,
            "cpu_baseline": cpu_line,
            "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "clocks": clk, "gpu_launches": gpu_launches, "version": sinn.version()}
    if graphs is not None:
        line["graph"] = ("each timed step = one replay of a CUDA graph captured around the SINN_SEARCH_NOSYNC search "
                         "(kernels / roofline from the same steps issued directly after the timed region)")
    if args.containers:  # F3: bitmap containers — index composition and the id bytes a batch reads
        st = G.stats()
        ids_entries = float(np.mean([a["ids"] for a in alg]))
        # the container terms are the index's most frequent terms, which every 1,024-query batch holds:
        # a batch reads their containers (8 B each) instead of one 4 B id per posting
        ids_cont = ids_entries - 4.0 * st["container_postings"] + 8.0 * st["containers"]
        line["containers"] = {"containers": st["containers"], "container_postings": st["container_postings"],
                              "postings": st["postings"], "ids_bytes_per_batch_entries_only": ids_entries,
                              "ids_bytes_per_batch_with_containers": ids_cont,
                              "ids_ratio": ids_cont / ids_entries if ids_entries > 0 else None}
        line["config"]["workload"] += "; bitmap containers (SINN_BITMAP_CONTAINERS)"
    G.close()
    del G
    gc.collect()
    torch.cuda.synchronize()
    return line


def sinn_score_kernel_name(cfg):
    return "k_doc_score (full pass: S1 walk + decode + accumulate + S2 threshold; + k_emit_rows for the sampled tiles when the sample kept its rows)"


def run_streaming(args, cfg, table, dev, stream, G, ws, rank):
    """configs[3]: grow 0 -> N in insert batches; after each insert delete floor(1% of live) random
    live ids and search one fresh batch.  Recycled ids are reused first (LIFO), then fresh ids
    (DESIGN.md input recipe).  Every phase is timed with CUDA events on the launching stream."""
    import torch
    import paper_2301_10622_b200 as sinn
    cap = cfg.N + cfg.insert_batch
    live = np.zeros(cap, bool)
    free: list[int] = []
    next_id = 0
    gen = 0
    rounds = []
    ins_ms_tot = del_ms_tot = srch_ms_tot = e2e_ms_tot = 0.0
    nq_tot = h2d_tot = 0
    hout = (np.empty((cfg.batch, cfg.k), np.uint32), np.empty((cfg.batch, cfg.k), np.float32))
    out = (torch.empty((cfg.batch, cfg.k), dtype=torch.int32, device=dev),
           torch.empty((cfg.batch, cfg.k), dtype=torch.float32, device=dev))

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    mean_nnz = float(np.diff(datagen.docs(cfg, 0, 20_000)[0]).mean())
    # capacity planning for the whole run (sinn_reserve): the raw store keeps a deleted row's entries
    # until its id is re-inserted, so it must hold every row inserted over the run (~N / 0.99^k rows
    # with 1 % deleted per round), not just the live ones; without this one growth of the multi-GB
    # raw store lands inside a timed insert round
    rows_total = 0
    live_n = 0
    while live_n < cfg.N:
        rows_total += cfg.insert_batch
        live_n += cfg.insert_batch
        live_n -= live_n // 100
    G.reserve(cap, int(rows_total * mean_nnz * 1.05))
    torch.cuda.synchronize()
    library_warmup(cfg, table, dev, args.bf16)
    torch.cuda.synchronize()
    G.profile(True)
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    rnd = 0
    prev_prof = None
    while live.sum() < cfg.N:
        B = cfg.insert_batch
        ip, ix, v = datagen.docs(cfg, gen, B)
        gen += B
        take = min(len(free), B)
        ids = np.empty(B, np.uint32)
        for r in range(take):
            ids[r] = free.pop()
        ids[take:] = np.arange(next_id, next_id + B - take, dtype=np.uint32)
        next_id += B - take
        t = (torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), torch.from_numpy(v).to(dev),
             torch.from_numpy(ids.view(np.int32)).to(dev))
        ins = timed(lambda: G.insert(*t))
        cur_prof = G.profile_read()  # (outside every timed region) per-phase device time of this insert
        ins_phases = {p_: round(cur_prof[p_][0] - (prev_prof[p_][0] if prev_prof else 0.0), 4)
                      for p_ in ("validate", "sketch", "postings", "raw")}
        live[ids] = True
        pool = np.flatnonzero(live).astype(np.uint32)
        dele = datagen.choose(pool, pool.size // 100, cfg.seed, rnd)
        td = torch.from_numpy(dele.view(np.int32)).to(dev)
        dl = timed(lambda: G.delete(td)) if dele.size else 0.0
        live[dele] = False
        free.extend(int(i) for i in dele)
        qp, qi, qv = datagen.queries(cfg, (rank * 10_000 + rnd) * cfg.batch, cfg.batch)
        tq = (torch.from_numpy(qp).to(dev), torch.from_numpy(qi).to(dev), torch.from_numpy(qv).to(dev))
        G.search(*tq, cfg.k, cfg.kprime, cfg.rerank, out=out)  # warm (workspace sizes for this index)
        sm = timed(lambda: G.search(*tq, cfg.k, cfg.kprime, cfg.rerank, out=out))  # synchronous call
        # end to end through the C ABI with HOST buffers: the round's queries copied in, results out
        e2e_ms_tot += timed(lambda: G.search_host(qp, qi, qv, cfg.k, cfg.kprime, cfg.rerank, out=hout))
        h2d_tot += qp.nbytes + qi.nbytes + qv.nbytes
        n_live = int(live.sum())
        rounds.append({"live": n_live, "insert_docs_per_s": B / (ins / 1e3), "insert_ms": ins, "delete_ms": dl,
                       "deleted": int(dele.size), "qps": cfg.batch / (sm / 1e3), "insert_phases_ms": ins_phases})
        prev_prof = G.profile_read()
        ins_ms_tot += ins
        del_ms_tot += dl
        srch_ms_tot += sm
        nq_tot += cfg.batch
        rnd += 1
    clk = clocks.stop()
    prof = G.profile_read()
    G.profile(False)
    qps = nq_tot * ws / (srch_ms_tot / 1e3)
    # the CPU oracle baseline on a bounded sample: the oracle over the first --cpu-sample-docs documents
    # of the stream (inserts only), 64 queries; QPS scaled by documents held / final live documents
    cpu_line = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        O, D, t_ins = oracle_sample_index(cfg, table, cpu_sample_docs(args, cfg), args.bf16)
        n_live = int(live.sum())
        qp, qi, qv = datagen.queries(cfg, 0, 64)
        t0 = time.perf_counter()
        O.search(qp, qi, qv, cfg.k, cfg.kprime, cfg.rerank, oracle.default_threads())
        cpu_s = time.perf_counter() - t0
        scale = D / max(n_live, 1)
        cpu_line = {"value": 64 / cpu_s * scale, "unit": "queries/s", "cores": oracle.default_threads(), "kind": "oracle",
                    "sample": f"64 queries over the first {D:,} documents of the stream (inserts only), QPS x {scale:.3g} "
                              f"(per-query work is proportional to the documents held; {n_live:,} live at the end)",
                    "insert_docs_per_s": D / t_ins}
        del O
    if rank == 0:
        line = {"metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": ws, "steps": rnd, "warmup": 0,
                "ms_per_step": srch_ms_tot / rnd, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_desc(cfg, args.bf16), "batch": cfg.batch, "k": cfg.k, "kprime": cfg.kprime,
                           "rerank": cfg.rerank, "rounds": rnd, "delete_basis": "1% of live",
                           "l2": "index > 1 GB from round 3 on; no flush"},
                "insert": {"value": cfg.insert_batch * rnd / (ins_ms_tot / 1e3), "unit": "docs/s",
                           "round_ms": [round(r["insert_ms"], 3) for r in rounds]},
                "delete_ms_per_round": del_ms_tot / rnd,
                "cpu_baseline": cpu_line,
                "e2e": {"value": nq_tot * ws / (e2e_ms_tot / 1e3), "unit": "queries/s",
                        "h2d_bytes_per_step": int(h2d_tot / max(rnd, 1)), "d2h_bytes_per_step": cfg.batch * cfg.k * 8,
                        "note": "every round's query batch searched again through sinn_search_host (host buffers)"},
                "curve": rounds[:: max(1, rnd // 12)] + [rounds[-1]],
                "kernels": {p: {"ms_total": prof[p][0], "launches": prof[p][2]} for p in prof},
                "clocks": clk, "gpu_launches": int(sum(prof[p][2] for p in prof)), "version": sinn.version()}
        print(json.dumps(line), flush=True)
    G.close()
    return 0


def run_sharded(args, cfg, ws, rank, local, dev, stream) -> int:
    """--shard: rank r holds the documents with id % ws == r (local id id // ws) and every rank searches the
    same query batches through sharded.ShardedIndex (stage 1 -> all-gather -> merge -> owner re-rank ->
    all-gather -> merge).  value = queries / max-rank time: strong scaling (the index is fixed, each GPU
    walks 1/ws of it)."""
    import torch
    import torch.distributed as dist

    import paper_2301_10622_b200 as sinn
    from paper_2301_10622_b200.sharded import ShardedIndex, route_rows_host

    table = datagen.hash_table(cfg)
    G = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=args.bf16, containers=args.containers)
    S = ShardedIndex(G, rank=rank, world=ws)
    mean_nnz = float(np.diff(datagen.docs(cfg, 0, min(cfg.N, 20_000))[0]).mean())
    G.reserve(cfg.N // ws + 1, int(cfg.N / ws * mean_nnz * 1.05))
    ins_ms, mine = 0.0, 0
    for s0 in range(0, cfg.N, cfg.insert_batch):
        c = min(cfg.insert_batch, cfg.N - s0)
        ip, ix, v = datagen.docs(cfg, s0, c)
        p, jx, w, lid = route_rows_host(ip, ix, v, np.arange(s0, s0 + c, dtype=np.uint32), ws, rank)  # host routing
        t = (torch.from_numpy(p).to(dev), torch.from_numpy(jx).to(dev), torch.from_numpy(w).to(dev),
             torch.from_numpy(lid.view(np.int32)).to(dev))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        G.insert(*t)
        e1.record(stream)
        torch.cuda.synchronize()
        ins_ms += e0.elapsed_time(e1)
        mine += lid.size
    ins_ms = max_over_ranks(ins_ms, ws, dev)
    nb = min(args.steps + args.warmup, 16)
    batches = []
    for b in range(nb):  # the SAME batches on every rank
        qp, qi, qv = datagen.queries(cfg, query_batch_start(0, nb, b, cfg.batch), cfg.batch)
        batches.append((torch.from_numpy(qp).to(dev), torch.from_numpy(qi).to(dev), torch.from_numpy(qv).to(dev)))
    res = None
    for t in range(args.warmup):
        res = S.search(*batches[t % nb], cfg.k, cfg.kprime, cfg.rerank)
    torch.cuda.synchronize()
    same = None
    if ws == 1 and res is not None:  # one shard: the protocol must return the plain search's ids
        pi, _ = G.search(*batches[(args.warmup - 1) % nb], cfg.k, cfg.kprime, cfg.rerank)
        same = float((pi == res[0]).float().mean().item())
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    G.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(args.steps):
        S.search(*batches[(args.warmup + t) % nb], cfg.k, cfg.kprime, cfg.rerank)
    e1.record(stream)
    torch.cuda.synchronize()
    el_ms = max_over_ranks(e0.elapsed_time(e1), ws, dev)
    prof = G.profile_read()
    G.profile(False)
    clk = clocks.stop()
    if ws > 1:
        dist.barrier()
    launches = int(sum(x[2] for x in prof.values())) + (2 if cfg.rerank else 1) * args.steps  # + the merges
    line = {"metric": METRIC, "value": cfg.batch * args.steps / (el_ms / 1e3), "unit": "queries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg, args.bf16), "batch": cfg.batch, "k": cfg.k, "kprime": cfg.kprime,
                       "rerank": cfg.rerank, "l2": l2_note(cfg),
                       "parallelism": f"document shards x{ws} (id % W), every rank scores the whole batch; one "
                                      f"all-gather of B*k'*8 B candidates and one of B*k*8 B winners per batch"},
            "exchange_bytes_per_step_per_gpu": cfg.batch * 8 * (cfg.kprime + (cfg.k if cfg.rerank else 0)),
            "insert": {"value": cfg.N / (ins_ms / 1e3), "unit": "docs/s", "docs_on_rank0": mine},
            "kernels": {name: {"ms_per_step": ms / args.steps, "launches_per_step": ln / args.steps}
                        for name, (ms, _, ln) in prof.items() if ln},
            "one_shard_ids_equal_plain_search": same, "clocks": clk, "gpu_launches": launches,
            "version": sinn.version()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: start the N ranks through torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_sinn(args)


if __name__ == "__main__":
    sys.exit(main())
