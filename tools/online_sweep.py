"""configs[4]-style online request-rate sweep on one B200: Poisson arrivals at
a fraction of the calibrated max throughput, served by the batch-size
controller (paper_1209_0410_b200/controller.py) over two CUDA streams;
prints one JSON line per load point with p50/p99 response time and the batch
size distribution (SPEC.md:456,504 metrics: mean/p99/throughput).

    python tools/online_sweep.py [--n 10000000] [--queries 200000]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.controller import BatchController, CudaBackend, Policy, poisson_arrivals, spin_idle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--queries", type=int, default=200_000)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--depth", type=int, default=350)
ap.add_argument("--max-batch", type=int, default=8192)
ap.add_argument("--loads", default="0.05,0.2,0.4,0.6,0.8,1.0")
a = ap.parse_args()

rows = H.gen_rows(0, a.n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
queries = H.gen_queries(0, a.queries, a.n)


def search(q, out, stream):
    ix.search_batch(q, a.k, a.depth, stream=stream, out=out)


def serve(arrivals, policy):
    be = CudaBackend(search, queries, a.k, slots=policy.slots, max_batch=policy.max_batch)
    clock = be.begin()
    return BatchController(policy).run(arrivals, be, clock=clock, idle=spin_idle(clock))


pol = Policy(max_batch=a.max_batch)
serve(np.zeros(min(a.queries, 50000)), pol)  # warm-up
sat = serve(np.zeros(a.queries), pol).summary()  # calibrate_max_throughput
qmax = sat["throughput_qps"]
print(json.dumps({"load": "saturation", **sat}), flush=True)
for f in [float(x) for x in a.loads.split(",")]:
    arr = poisson_arrivals(f * qmax, a.queries, seed=1)
    s = serve(arr, pol).summary()
    print(json.dumps({"load_fraction": f, "offered_qps": f * qmax, **s}), flush=True)
