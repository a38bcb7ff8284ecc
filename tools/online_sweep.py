"""configs[4]: online request-rate sweep on the C++ batch-size controller
(libhcg hcg_server_*, csrc/serve.cpp; DTAHE Alg. 3 without the CPU branch).

One process drives G GPUs: G = 1 serves one index; G > 1 a shard group
(shard r = ids r, r+G, ... built on GPU r from the generator, per-shard depth
from the planner; NCCL all-gather + merge inside the library).  Queries live
in host memory and arrive open-loop (Poisson) at fractions of
the calibrated max throughput (all arrivals at t = 0); every
response time includes the query's H2D and its results' D2H.  One JSON line
per load point (p50 / p99 / mean response time, throughput, batch sizes).

    python tools/online_sweep.py --gpus 1              # 10M on one GPU
    python tools/online_sweep.py --gpus 4 --rows 100000000
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.controller import poisson_arrivals  # noqa: E402
from paper_1209_0410_b200.server import Server, latency_summary  # noqa: E402
from paper_1209_0410_b200.sharded import ShardGroup, shard_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--rows", type=int, default=0, help="rows (default 10M on 1 GPU, 100M sharded)")
ap.add_argument("--queries", type=int, default=200_000)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--depth", type=int, default=350)
ap.add_argument("--max-batch", type=int, default=8192)
ap.add_argument("--min-batch", type=int, default=1)
ap.add_argument("--max-wait-us", type=float, default=0.0)
ap.add_argument("--loads", default="0.05,0.2,0.4,0.6,0.8,1.0")
ap.add_argument("--slots", type=int, default=2, help="batches in flight (2 = double buffer)")
ap.add_argument("--check", type=int, default=2000, help="queries of the saturation run re-checked against hcg_search")
a = ap.parse_args()

G = a.gpus
n = a.rows or (10_000_000 if G == 1 else 100_000_000)
scheme = H.default_scheme(128, 8, 16)
t0 = time.time()
if G == 1:
    target = H.MulticurvesIndex(H.gen_rows(0, n, device=0), scheme, H.LIFTED, device=0)
    depth = a.depth
else:
    shards = []
    for r in range(G):
        torch.cuda.set_device(r)
        rows = H.gen_rows(r, shard_rows(n, r, G), stride=G, device=r)
        shards.append(H.MulticurvesIndex(rows, scheme, H.LIFTED, device=r, id_base=r, id_stride=G))
        del rows
        torch.cuda.synchronize(r)
    torch.cuda.set_device(0)
    target = ShardGroup.adopt(shards)
    depth = H.shard_probe_depth(a.depth, G)
build_s = time.time() - t0
queries = H.gen_queries(0, a.queries, n, device=0).cpu().numpy()
srv = Server(target, a.k, depth, max_batch=a.max_batch, min_batch=a.min_batch, max_wait=a.max_wait_us * 1e-6,
             slots=a.slots)
head = {"gpus": G, "n": n, "depth": a.depth, "shard_depth": depth, "k": a.k, "max_batch": a.max_batch,
        "min_batch": a.min_batch, "max_wait_us": a.max_wait_us, "slots": a.slots, "build_s": round(build_s, 1),
        "server": "C++ hcg_server (csrc/serve.cpp), host queries in / host results out"}


def run(arrivals):
    ids, sq, ln, lat, sizes = srv.replay(queries[:len(arrivals)], arrivals)
    makespan = float(np.max(arrivals + lat) - arrivals[0])
    return latency_summary(lat, sizes, makespan), (ids, sq, ln)


run(np.zeros(min(a.queries, 50_000)))  # warm-up
sat, (ids, sq, ln) = run(np.zeros(a.queries))  # calibrate_max_throughput
# the served results are the search's results
c = min(a.check, a.queries)
if G == 1:
    ri, rs, rl = target.search_batch(queries[:c], a.k, depth)
else:
    ri, rs, rl = target.search(queries[:c], a.k, depth)
sat["results_identical_to_direct_search"] = bool(np.array_equal(ids[:c], ri) and np.array_equal(sq[:c], rs)
                                                 and np.array_equal(ln[:c], rl))
qmax = sat["throughput_qps"]
print(json.dumps({**head, "load": "saturation", **sat}), flush=True)
for f in [float(x) for x in a.loads.split(",") if x]:
    s, _ = run(poisson_arrivals(f * qmax, a.queries, seed=1))
    print(json.dumps({**head, "load_fraction": f, "offered_qps": f * qmax, **s}), flush=True)
srv.close()
