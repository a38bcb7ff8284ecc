"""Probe: does processing a batch in curve-0 rank order (neighbouring queries
share candidate rows while they are in flight) cut the gather's DRAM traffic?
Times search_timed on the generator's query order and on the same queries
sorted by their curve-0 rank."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D = 10_000_000, 100_000, 10, 350
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = [H.gen_queries(b * Q, Q, n) for b in range(4)]
sorted_qs = []
for q in qs:
    r, _, _ = ix.windows(q.cpu().numpy(), D)
    order = torch.from_numpy(np.argsort(r[:, 0], kind="stable").astype(np.int64)).cuda()
    sorted_qs.append(q[order].contiguous())
out = (torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
       torch.empty((Q,), dtype=torch.uint32, device="cuda"))
for name, batch in (("generator order", qs), ("curve-0 rank order", sorted_qs)) * 2:
    for b in range(2):
        ix.search_timed(batch[b], k, D, out=out)
    t = [ix.search_timed(batch[b % 4], k, D, out=out) for b in range(6)]
    med = [sorted(x[i] for x in t)[3] for i in range(3)]
    print(f"{name}: locate {med[0]:.3f} union {med[1]:.3f} gather {med[2]:.3f} ms", flush=True)
