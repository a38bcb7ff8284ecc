#!/usr/bin/env python3
"""bench.py -- Hypercurves approximate-kNN hot path on B200 (BASELINE.json).

One "step" = one batched search of a fresh batch of synthetic queries through
the whole hot path (per-curve keys -> lower_bound -> windows -> dedup ->
gather -> exact L2 -> top-k; at N>1 also the routed exchange + merge).

  N=1 : configs[1] -- 10M x 128-d uint8 (synthetic SIFT-like),
        100K queries per step, k=10, 8 Hilbert curves, probe depth 350,
        lifted view (1 + b/256, m=16; recall@10 ~0.99).
  N>1 : configs[2] -- 100M x 128-d sharded id mod N over N ranks (one process
        per GPU, torchrun), per-shard depth from the equivalence planner
        (miss < 2%); the packed top-k lists are routed to
        their aggregator rank (route_to_aggregator: NCCL
        send / recv of 1/N query blocks inside libhcg) and merged by K4.

value   : queries/s with queries already resident in HBM (device timed,
          CUDA events, max over ranks).
e2e     : the same through the public API with pinned HOST query buffers and a
          host read-back of every step's results (H2D + D2H inside the timing).
roofline: the refine kernel (gather + L2 + top-k) -- algorithmic bytes per
          launch / its CUDA-event duration vs the measured HBM copy peak.
cpu_baseline : the reference's CPU path (oracle/_ref: the reference's own
          curve.cpp + vecio.cpp + the multicurves.hpp restatement) on this
          host's cores, over a bounded query sample of the same workload.

--impl reference runs only that CPU reference path (rank 0; other ranks exit).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "kNN queries/sec at fixed probe depth & recall@10, 1/2/4/8 B200; HBM GB/s"
DATA = "synthetic: SURVEY.md §8(d) counter-based SIFT-like uint8 generator (same bytes on CPU and GPU)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--rows", "--n", dest="n", type=int, default=0,
                   help="database rows (default 10M at N=1, 100M at N>1); spell it --rows under torchrun")
    p.add_argument("--queries", type=int, default=100_000, help="queries per step")
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--depth", type=int, default=350)
    p.add_argument("--curves", type=int, default=8)
    p.add_argument("--view", choices=["lifted", "raw"], default="lifted")
    p.add_argument("--kind", choices=["hilbert", "zorder"], default="hilbert")
    p.add_argument("--shard-depth", default="planned",
                   help="N>1 per-shard depth: planned | full | optimist | <int>")
    p.add_argument("--recall-sample", type=int, default=1000)
    p.add_argument("--cpu-sample", type=int, default=100_000,
                   help="queries of step 0 in our arm's CPU baseline + parity sample (~10 s on 16 cores)")
    p.add_argument("--ref-sample", type=int, default=100_000,
                   help="queries per step timed by the reference arm (--impl reference); default = a whole step")
    p.add_argument("--cert-sample", type=int, default=200,
                   help="queries of step 0 certified against the reference semantics (oracle/certify.py)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--latency-batches", default="1,16,256,4096,65536")
    p.add_argument("--latency-reps", type=int, default=20)
    return p.parse_args()


# --------------------------------------------------------------- plumbing ----
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[6]) or 0) > 0] or self.rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(self.rows[0][1]), "reasons": reasons, "samples": len(self.rows),
                "samples_under_load": len(loaded)}


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_key: str):
    """dram bytes per refine launch from a committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "refine_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(config_key)
        return e if e else None
    except Exception:
        return None


# --------------------------------------------------------- CPU reference ----
def cpu_reference_qps(rows_u8, queries_u8, curves, m, kind, view, k, depth, threads, reps=1):
    """The reference's CPU path (oracle/_ref) on a bounded query sample; returns
    (q/s, seconds, results of the last rep)."""
    from oracle import pyoracle as P
    ri = P.RefIndex(rows_u8, curves, m, kind, view)
    best = None
    res = None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = ri.search(queries_u8, k, depth, threads=threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    del ri
    return queries_u8.shape[0] / best, best, res


def workload_name(n_total: int, Q: int, k: int, C: int, D: int, world: int) -> str:
    base = f"{n_total / 1e6:g}M x 128-d, {Q} queries/step, k={k}, {C} curves, probe depth {D}"
    if n_total >= 100_000_000:
        tag = ("configs[2]: 100M sharded id mod N over N GPUs (hcg_shard_group: per-shard search, routed NCCL "
               "exchange of 1/N query blocks, K4 merge)" if world > 1 else "configs[2] at N=1: 100M on one B200 (same-workload anchor)")
    elif n_total == 10_000_000 and world == 1:
        tag = "configs[1]"
    elif n_total == 1_000_000:
        tag = "configs[0]"
    else:
        tag = "custom" if world == 1 else "sharded id mod N"
    return f"{tag}: {base}"


# ------------------------------------------------------------------- ours ----
def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_1209_0410_b200 as H
    from paper_1209_0410_b200.sharded import ShardedIndex, recall

    rank, world, local = dist_env()
    if world != a.gpus:
        a.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    view = H.LIFTED if a.view == "lifted" else H.RAW
    m = 16 if a.view == "lifted" else 8
    kind = H.HILBERT if a.kind == "hilbert" else H.ZORDER
    n_total = a.n or (10_000_000 if world == 1 else 100_000_000)
    Q, k, D, C = a.queries, a.k, a.depth, a.curves
    if world == 1:
        shard_depth = D
    elif a.shard_depth == "planned":
        shard_depth = H.shard_probe_depth(D, world, 0.02)
    elif a.shard_depth == "full":
        shard_depth = D
    elif a.shard_depth == "optimist":
        shard_depth = 2 * (((D + 1) // 2 + world - 1) // world)
    else:
        shard_depth = int(a.shard_depth)
    scheme = H.default_scheme(128, C, m, kind)

    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    sidx = ShardedIndex.from_generator(n_total, scheme, view, rank, world, local)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    if world > 1:
        dist.barrier()

    # the sampler starts here so that nvidia-smi is up before the timed region
    # without idling the GPU (an idle gap lets the SM clock drop)
    clocks = ClockSampler(local)
    clocks.start()
    nb = a.warmup + a.steps
    batches = [H.gen_queries(b * Q, Q, n_total, device=local) for b in range(nb)]
    out = (torch.empty((Q, k), dtype=torch.uint64, device=dev),
           torch.empty((Q, k), dtype=torch.uint32, device=dev),
           torch.empty((Q,), dtype=torch.uint32, device=dev))

    # N>1: the aggregate is routed (route_to_aggregator):
    # each rank merges the partials of its own 1/N block of the batch, so the
    # box's ranks together hold every query's global top-k
    routed = world > 1
    block = [0, Q]

    def search_step(q, out_):
        if routed:
            _, block[0], block[1] = sidx.shard_group.search_routed(q, k, shard_depth, out=out_)
            return block[0], block[0] + block[1]
        sidx.search(q, k, shard_depth, out=out_)
        return 0, int(q.shape[0])

    def step(b):
        search_step(batches[b], out)

    launches = [0]  # our kernels launched inside the timed region (libhcg's counter)

    def timed(fn):
        for b in range(a.warmup):
            fn(b)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n0 = H.lib().hcg_launch_count()
        e0.record(stream)
        for s in range(a.steps):
            fn(a.warmup + s)
        e1.record(stream)
        launches[0] = H.lib().hcg_launch_count() - n0
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    ms_total = timed(step)

    # e2e: pinned host queries in, pinned host results out, every step, through
    # the public API (HostPipeline: H2D of step b+1 and D2H of step b overlap
    # the search of step b; each step's copies stay inside the timed region).
    from paper_1209_0410_b200.pipeline import HostPipeline
    host_batches = [bt.cpu().pin_memory() for bt in batches]
    host_outs = [(torch.empty((Q, k), dtype=torch.uint64).pin_memory(),
                  torch.empty((Q, k), dtype=torch.uint32).pin_memory(),
                  torch.empty((Q,), dtype=torch.uint32).pin_memory()) for _ in range(2)]
    pipe = HostPipeline(search_step, k, Q, device=local)
    pipe.run(host_batches[:a.warmup], [host_outs[b % 2] for b in range(a.warmup)])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    pipe.run(host_batches[a.warmup:], [host_outs[b % 2] for b in range(a.steps)], e0, e1)
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    clocks.stop()
    h2d = Q * 128
    rows_back = block[1] if routed else Q  # each rank reads back the rows it aggregated
    d2h = rows_back * (k * 8 + k * 4 + 4)

    # dominant-kernel roofline (outside the timed region): per-launch device
    # times of locate / candidate union / gather+score, CUDA events on `stream`.
    tl, tu, tg = [], [], []
    for b in range(a.warmup, nb):
        ml, mu, mg = sidx.local.search_timed(batches[b], k, shard_depth, out=out)
        tl.append(ml)
        tu.append(mu)
        tg.append(mg)
    U = sidx.local.candidate_counts(batches[a.warmup], shard_depth).astype(np.float64)
    take = min(shard_depth, sidx.local.size())
    # Which K3c runs (the library's dispatch, search.cu refine_dispatch): for
    # k <= 128 and batches >= 16K on a reordered index the union is skipped and
    # k_gather_nu walks the windows; otherwise k_union_reg + k_gather.
    unionless = sidx.local.unionless(Q, k, shard_depth)
    if unionless:
        # k_gather_nu reads the C windows of ids, each unique row once (repeats
        # reached through a second curve are re-reads, not algorithmic), the
        # query, and writes k (id, sqdist) pairs + len.
        bytes_gather = float(U.sum() * 128 + Q * (4 * C * take + 4 * C + 128 + 12 * k + 4))
        bytes_union = 0.0
    else:
        # k_gather reads each unique row (128 B) + its list entry (4 B), the query
        # (128 B) and the count, and writes k (id, sqdist) pairs + len.
        bytes_gather = float(U.sum() * (128 + 4) + Q * (128 + 4 + 12 * k + 4))
        # k_union reads C windows of ids + C begins and writes the unique list.
        bytes_union = float(Q * (4 * C * take + 4 * C) + U.sum() * 4)
    gather_ms = statistics.median(tg)
    union_ms = statistics.median(tu)
    peak, peak_src = measured_peak_gbs()
    achieved = bytes_gather / (gather_ms * 1e-3) / 1e9
    logn = max(1, int(np.ceil(np.log2(max(2, sidx.local.size())))))
    bytes_q = float(U.mean() * 128 + 4 * C * take + 16 * C * logn + 128 + 8 * k)

    # recall@k on a query sample against exact brute force (GPU K5, merged across shards).
    rs = min(a.recall_sample, Q)
    qs = batches[0][:rs].contiguous()
    got = sidx.search(qs, k, shard_depth)
    exact = sidx.brute_force(qs, k)
    rec = recall(got[0].cpu().numpy(), exact[0].cpu().numpy(), k)

    # latency per batch size (device-resident queries and results, one call of
    # the C entry point -- hcg_search, or hcg_shard_group_search at N>1 -- per
    # sample: CUDA events on the stream around the call, so its host-side work
    # counts; Python argument marshalling is done once, outside)
    lat = {}
    L = H.lib()
    for bs in [int(x) for x in a.latency_batches.split(",") if x]:
        if bs > Q:
            continue
        qb = batches[0][:bs].contiguous()
        o = (torch.empty((bs, k), dtype=torch.uint64, device=dev),
             torch.empty((bs, k), dtype=torch.uint32, device=dev),
             torch.empty((bs,), dtype=torch.uint32, device=dev))
        ptrs = (qb.data_ptr(), bs, k, shard_depth, o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(), stream.cuda_stream)
        if world > 1:
            call = lambda: L.hcg_shard_group_search(sidx.shard_group._h, *ptrs)  # noqa: E731
        else:
            call = lambda: L.hcg_search(sidx.local._h, *ptrs)  # noqa: E731
        for _ in range(3):
            assert call() == 0, L.hcg_last_error()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.latency_reps):
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        lat[str(bs)] = {"p50_ms": round(ts[len(ts) // 2], 4), "p99_ms": round(ts[min(len(ts) - 1, int(0.99 * len(ts)))], 4),
                        "qps_at_p50": round(bs / (ts[len(ts) // 2] * 1e-3), 1)}

    # Certificate parity on a query sample (oracle/certify.py; every config,
    # every N): each rank recomputes its shard's top-k from the reference's
    # semantics -- oracle keys of the regenerated rows around every window,
    # lower bound, window rule, exact distances, (distance, id) order -- and
    # rank 0 merges the shards' lists and compares them with the GPU result.
    cert = None
    if a.cert_sample > 0:
        from oracle import certify as CE
        from oracle import pyoracle as P
        cs = min(a.cert_sample, Q)
        qc = batches[0][:cs].contiguous()
        gi, gs, gl = (x.cpu().numpy() for x in sidx.search(qc, k, shard_depth))
        part = CE.certify_shard(sidx.local, qc.cpu().numpy(), shard_depth, k, 1 if a.view == "lifted" else 0, m,
                                kind)
        parts = [part]
        if world > 1:
            parts = [None] * world if rank == 0 else None
            dist.gather_object(part, parts, dst=0)
        if rank == 0:
            oi, od, ol = P.merge_shard_lists([p_[:3] for p_ in parts], k)
            rooted = np.sqrt(gs.astype(np.float64)) * view.scale
            mism = sum(int(not (gl[q] == ol[q] and np.array_equal(gi[q, :ol[q]], oi[q, :ol[q]])
                               and rooted[q, :ol[q]].tobytes() == od[q, :ol[q]].tobytes())) for q in range(cs))
            failed = {}
            for p_ in parts:
                for key_, v in p_[3]["failed_checks"].items():
                    failed[key_] = failed.get(key_, 0) + v
            cert = {"sample_queries": cs, "shards": world, "rows_per_shard": [p_[3]["rows"] for p_ in parts],
                    "failed_checks": failed, "mismatched_queries": mism,
                    "identical": bool(mism == 0 and sum(failed.values()) == 0),
                    "method": "oracle/certify.py: oracle keys of the regenerated rows at every window's sorted "
                              "positions (order, lower bound, window rule), exact distances of the candidate union, "
                              "(distance, id) top-k per shard, merged"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and n_total <= 20_000_000 and not a.no_cpu_baseline:
        threads = os.cpu_count() or 1
        S = min(a.cpu_sample, Q)
        rows_h = H.gen_rows(0, n_total, device=local).cpu().numpy()
        qh = batches[0][:S].cpu().numpy()
        qps_cpu, secs, (rids, rdist, rln) = cpu_reference_qps(rows_h, qh, C, m, kind, 1 if a.view == "lifted" else 0,
                                                             k, D, threads)
        del rows_h
        gi, gs, gl = sidx.local.search_batch(qh, k, D)
        same = (np.array_equal(gl, rln) and np.array_equal(gi, rids)
                and np.array_equal(sidx.local.rooted(gs), rdist))
        parity = {"sample_queries": S, "ids_and_distances_identical": bool(same)}
        from oracle import pyoracle as P
        cpu = {"value": round(qps_cpu, 1), "unit": "queries/s", "cores": threads,
               "kind": "reference" if P.ref_available() else "port",
               "sample": f"{S} queries of step 0's batch over the same {n_total} rows "
                         f"(reference curve.cpp/vecio.cpp + multicurves.hpp restatement, "
                         f"{threads} threads, {secs:.2f} s wall)"}

    if rank == 0:
        ms_step = ms_total / a.steps
        value = Q * a.steps / (ms_total * 1e-3)
        e2e_value = Q * a.steps / (ms_e2e * 1e-3)
        traffic = ncu_traffic(f"k{k}_Q{Q}_D{shard_depth}_{a.view}_n{sidx.local.size()}")
        line = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": "queries/s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None,
            "dtype": "u8",
            "data": DATA,
            "config": {
                "workload": workload_name(n_total, Q, k, C, D, world),
                "n_db": n_total, "queries_per_step": Q, "k": k, "curves": C, "probe_depth": D,
                "shard_probe_depth": shard_depth, "curve": a.kind, "view": a.view, "bits_per_dim": m,
                "recall_at_k": round(rec, 4), "recall_sample": rs,
                "l2": "inputs larger than L2 (descriptors + sorted curves > 2.8 GB vs 126 MB L2); "
                      "a fresh query batch every step",
                "build_s": round(build_s, 3),
                "device_index_bytes": sidx.local.device_bytes(),
            },
            "roofline": {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": ("k_gather_nu (walk of the C windows + gather of their rows + exact L2 + top-k, "
                           "repeats dropped in the top-k; no separate union)" if unionless else
                           "k_gather (gather of the unique candidate rows + exact L2 + top-k)"),
                "algorithmic_bytes_per_launch": bytes_gather,
                "launch_ms": round(gather_ms, 4),
                # device time of the step's kernels (locate + batch order / union + refine), CUDA
                # events on the launching stream; ms_per_step minus this is launch gaps + (N>1) the
                # exchange and merge
                "kernel_ms_sum": round(statistics.median(tl) + union_ms + gather_ms, 4),
                "other_kernels_ms": ({"k_locate": round(statistics.median(tl), 4),
                                      "batch_order_sort": round(union_ms, 4)} if unionless else
                                     {"k_locate": round(statistics.median(tl), 4), "k_union": round(union_ms, 4)}),
                "k_union_algorithmic_gbs": (round(bytes_union / max(union_ms, 1e-9) / 1e6, 1)
                                            if not unionless else None),
                "peak_source": peak_src,
                "bytes_per_query_B_q": round(bytes_q, 1),
                "unique_candidates_per_query": round(float(U.mean()), 1),
                "step_hbm_gbs": round(Q * a.steps / (ms_total * 1e-3) * bytes_q / 1e9, 1),
                # frac can exceed 1: the algorithmic bytes count every candidate row as a
                # DRAM read, while rows stored and queried in curve-0 order are partly
                # served from L2 (see traffic); dram_gbs is the ncu DRAM traffic per launch
                # over this run's launch time
                "dram_gbs": (round(traffic["traffic_bytes"] / (gather_ms * 1e-3) / 1e9, 1)
                             if isinstance(traffic, dict) and traffic.get("traffic_bytes") else None),
            },
            "cpu_baseline": cpu,
            "parity_vs_reference": parity,
            "parity_certificate": cert,
            "e2e": {"value": round(e2e_value, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches[0]),
            "clocks": clocks.summary(),
            "latency": lat,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# -------------------------------------------------------------- reference ----
def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as P

    view = 1 if a.view == "lifted" else 0
    m = 16 if a.view == "lifted" else 8
    kind = 1 if a.kind == "hilbert" else 0
    n_total = a.n or (10_000_000 if world == 1 else 100_000_000)
    threads = os.cpu_count() or 1
    k, D, C = a.k, a.depth, a.curves
    if world == 1:
        rows = P.gen_rows(0, n_total, threads)
        depth = D
        note = f"{n_total} rows"
        shards_on_host = 1
    else:
        # The host must run every shard of the configs[2] partition; one shard
        # (capped at 12.5M rows, the N=8 shard size) is built and timed, and the
        # host throughput is that shard's rate divided by the shard count.
        from paper_1209_0410_b200.multicurves import shard_probe_depth  # pure host math
        cnt = min((n_total + world - 1) // world, 12_500_000)
        rows = P.gen_rows(0, cnt, threads, stride=world)
        depth = shard_probe_depth(D, world, 0.02) if a.shard_depth == "planned" else D
        note = f"shard 0 of {world} ({cnt} rows, per-shard depth {depth}); q/s = shard rate / {world}"
        shards_on_host = world
    t0 = time.perf_counter()
    ri = P.RefIndex(rows, C, m, kind, view)
    build_s = time.perf_counter() - t0
    S = min(a.ref_sample, a.queries)
    # warm-up steps on a 10K-query slice (caches and threads only), timed steps on the whole S
    steps_q = [P.gen_queries(b * a.queries, S if b >= a.warmup else min(S, 10_000), n_total, threads)
               for b in range(a.warmup + a.steps)]
    for b in range(a.warmup):
        ri.search(steps_q[b], k, depth, threads)
    t0 = time.perf_counter()
    for s in range(a.steps):
        ri.search(steps_q[a.warmup + s], k, depth, threads)
    dt = time.perf_counter() - t0
    value = S * a.steps / dt / shards_on_host
    kind_s = "reference" if P.ref_available() else "port"
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(dt / a.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": DATA,
        "config": {"workload": workload_name(n_total, a.queries, k, C, D, world), "n_db": n_total,
                   "queries_per_step_sample": S, "same_config_as_gpu_arm": S == a.queries, "k": k, "curves": C, "probe_depth": D,
                   "shard_probe_depth": depth, "view": a.view, "bits_per_dim": m, "curve": a.kind,
                   "build_s": round(build_s, 2)},
        "cpu_baseline": {"value": round(value, 1), "unit": "queries/s", "cores": threads, "kind": kind_s,
                         "sample": f"{S} queries per step over {note}; reference curve.cpp/vecio.cpp + "
                                   f"multicurves.hpp restatement, query-parallel on {threads} threads"},
        "e2e": {"value": round(value, 1), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line on the original stdout (everything else -- NCCL's
    version banner included -- was redirected to stderr in main())."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # One JSON line on stdout: native libraries (NCCL prints its version with
    # printf at communicator init) write to fd 1 directly, so move fd 1 to
    # stderr for the run and keep a private handle on the real stdout.
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
