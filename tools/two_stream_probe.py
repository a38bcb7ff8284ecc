"""Do consecutive 100K-query batches gain from two streams (the next batch's
locate / batch order filling the tail of the previous gather)?  10M lifted,
k=10, depth 350: 10 steps on one stream vs alternating two streams."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D, S = 10_000_000, 100_000, 10, 350, 10
ix = H.MulticurvesIndex(H.gen_rows(0, n), H.default_scheme(128, 8, 16), H.LIFTED)
batches = [H.gen_queries(b * Q, Q, n) for b in range(S + 3)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
outs = [(torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
         torch.empty((Q,), dtype=torch.uint32, device="cuda")) for _ in range(2)]


def run(nstreams):
    for b in range(3):
        ix.search_batch(batches[b], k, D, out=outs[0], stream=streams[0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for s in range(S):
        i = s % nstreams
        ix.search_batch(batches[3 + s], k, D, out=outs[i], stream=streams[i])
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    e1.synchronize()
    return e0.elapsed_time(e1) / S


for rep in range(3):
    for ns in (1, 2):
        ms = run(ns)
        print(json.dumps({"streams": ns, "ms_per_step": round(ms, 4), "qps": round(Q / ms * 1e3)}), flush=True)
