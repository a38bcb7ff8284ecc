"""configs[4]: online request-rate sweep.  Poisson arrivals at fractions of
the calibrated max throughput, served by the batch-size controller
(paper_1209_0410_b200/controller.py); one JSON line per load point with
p50/p99 response time, throughput and the batch-size distribution
(SPEC.md:456,504 metrics).

    python tools/online_sweep.py                              # 1 GPU, 10M
    torchrun --nproc-per-node 8 tools/online_sweep.py         # 100M sharded over 8
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.controller import (BatchController, CudaBackend, Policy, ShardedBackend,  # noqa: E402
                                             poisson_arrivals, spin_idle)
from paper_1209_0410_b200.sharded import ShardedIndex  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=0, help="rows (default 10M on 1 GPU, 100M sharded)")
ap.add_argument("--queries", type=int, default=200_000)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--depth", type=int, default=350)
ap.add_argument("--max-batch", type=int, default=8192)
ap.add_argument("--loads", default="0.05,0.2,0.4,0.6,0.8,1.0")
ap.add_argument("--slots", type=int, default=2, help="batches in flight (2 = double buffer)")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = a.n or (10_000_000 if world == 1 else 100_000_000)
sidx = ShardedIndex.from_generator(n, H.default_scheme(128, 8, 16), H.LIFTED, rank, world, local)
depth = a.depth if world == 1 else H.shard_probe_depth(a.depth, world)
queries = H.gen_queries(0, a.queries, n, device=local)


def search(q, out, stream=None):
    if world == 1:
        sidx.local.search_batch(q, a.k, depth, stream=stream, out=out)
    else:
        sidx.search(q, a.k, depth, out=out)


cmd_group = dist.new_group(backend="gloo") if world > 1 else None


def make_backend(pol):
    if world == 1:
        return CudaBackend(search, queries, a.k, slots=pol.slots, max_batch=pol.max_batch)
    return ShardedBackend(lambda q, out: search(q, out), queries, a.k, max_batch=pol.max_batch, slots=pol.slots,
                          cmd_group=cmd_group)


def serve(arrivals, pol):
    be = make_backend(pol)
    if rank != 0:
        be.follow()
        return None
    clock = be.begin()
    res = BatchController(pol).run(arrivals, be, clock=clock, idle=spin_idle(clock))
    if world > 1:
        be.stop()
    return res.summary()


pol = Policy(max_batch=a.max_batch, slots=a.slots)
serve(np.zeros(min(a.queries, 50000)), pol)  # warm-up
sat = serve(np.zeros(a.queries), pol)  # calibrate_max_throughput
qmax = torch.tensor([sat["throughput_qps"] if rank == 0 else 0.0], device=f"cuda:{local}")
if world > 1:
    dist.broadcast(qmax, 0)
qmax = float(qmax.item())
if rank == 0:
    print(json.dumps({"gpus": world, "n": n, "shard_depth": depth, "load": "saturation", **sat}), flush=True)
for f in [float(x) for x in a.loads.split(",")]:
    s = serve(poisson_arrivals(f * qmax, a.queries, seed=1), pol)
    if rank == 0:
        print(json.dumps({"gpus": world, "load_fraction": f, "offered_qps": f * qmax, **s}), flush=True)
if world > 1:
    dist.destroy_process_group()
