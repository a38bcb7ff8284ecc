"""configs[3]: probe-depth x curve-count sweep on 10M x 128-d (one B200),
recall@k vs queries/s for k=10 and k=100.  One JSON line per point.

    python tools/sweep.py [--n 10000000] [--queries 100000]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.sharded import recall  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--queries", type=int, default=100_000)
ap.add_argument("--depths", default="16,64,128,256,350,512,1024,4096")
ap.add_argument("--curves", default="2,4,8,16")
ap.add_argument("--ks", default="10,100")
ap.add_argument("--view", default="lifted")
ap.add_argument("--recall-sample", type=int, default=500)
a = ap.parse_args()
view, m = (H.LIFTED, 16) if a.view == "lifted" else (H.RAW, 8)
rows = H.gen_rows(0, a.n)
qs = H.gen_queries(0, a.queries, a.n)
sample = qs[:a.recall_sample].contiguous()
truth = {}
for C in [int(x) for x in a.curves.split(",")]:
    if (128 // C) * m > 1024:
        continue
    ix = H.MulticurvesIndex(rows, H.default_scheme(128, C, m), view)
    for k in [int(x) for x in a.ks.split(",")]:
        if k not in truth:
            truth[k] = ix.brute_force(sample, k)[0].cpu().numpy()
        out = (torch.empty((a.queries, k), dtype=torch.uint64, device="cuda"),
               torch.empty((a.queries, k), dtype=torch.uint32, device="cuda"),
               torch.empty((a.queries,), dtype=torch.uint32, device="cuda"))
        for D in [int(x) for x in a.depths.split(",")]:
            try:
                ix.search_batch(qs, k, D, out=out)  # warm-up
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    ix.search_batch(qs, k, D, out=out)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / 3
                got = ix.search_batch(sample, k, D)[0].cpu().numpy()
                U = float(ix.candidate_counts(qs[:2000], D).mean())
                print(json.dumps({"curves": C, "depth": D, "k": k, "view": a.view, "n": a.n,
                                  "qps": a.queries / (ms * 1e-3), "ms_per_batch": ms,
                                  "unionless": ix.unionless(a.queries, k, D),
                                  "recall_at_k": recall(got, truth[k], k), "unique_candidates": U}), flush=True)
            except Exception as e:  # capacity limits (curves x depth) are reported, not fatal
                print(json.dumps({"curves": C, "depth": D, "k": k, "error": str(e)}), flush=True)
    del ix
