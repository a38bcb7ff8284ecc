"""Probe: does storing the descriptors in curve-0 key order (clusters become
contiguous) speed up the candidate gather?  Times search on the generator's
order and on rows permuted by curve 0's sorted order (ids differ; timing only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D = 10_000_000, 100_000, 10, 350
scheme = H.default_scheme(128, 8, 16)
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, scheme, H.LIFTED)
perm = torch.from_numpy(ix.subindex(0).astype("int64")).cuda()
rows_p = rows[perm].contiguous()
ixp = H.MulticurvesIndex(rows_p, scheme, H.LIFTED)
del rows, rows_p
qs = [H.gen_queries(b * Q, Q, n) for b in range(4)]
out = (torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
       torch.empty((Q,), dtype=torch.uint32, device="cuda"))
for name, index in (("generator order", ix), ("curve-0 order", ixp), ("generator order", ix), ("curve-0 order", ixp)):
    for b in range(2):
        index.search_timed(qs[b], k, D, out=out)
    t = [index.search_timed(qs[b % 4], k, D, out=out) for b in range(6)]
    med = [sorted(x[i] for x in t)[3] for i in range(3)]
    print(f"{name}: locate {med[0]:.3f} union {med[1]:.3f} gather {med[2]:.3f} ms", flush=True)
