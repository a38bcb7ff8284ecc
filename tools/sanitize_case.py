"""Small end-to-end case for compute-sanitizer: build (keygen, radix sort),
search (locate, union, gather both variants), candidates, brute force, merge,
insert -- each kernel launched at least once on tiny inputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

rows = H.gen_rows(0, 3000)
qs = H.gen_queries(0, 300, 3000)
for view, m, C in ((H.LIFTED, 16, 8), (H.RAW, 8, 16)):
    ix = H.MulticurvesIndex(rows, H.default_scheme(128, C, m), view)
    ix.search_batch(qs, 10, 350)            # CTA gather (small batch)
    ix.search_batch(qs[:3], 100, 64)
    ix.candidates(qs[:4].cpu().numpy(), 64)
    ix.brute_force(qs[:16], 10)
    ix.insert(H.gen_rows(3000, 500))
    ix.search_batch(qs, 10, 4000)           # large candidate sets -> CAS union
big = H.gen_queries(0, 6000, 3000)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
ix.search_batch(big, 10, 350)               # warp-per-query gather
p = torch.stack([ix.search_packed(qs, 10, 64), ix.search_packed(qs, 10, 32)])
H.merge_packed(p, 10)
torch.cuda.synchronize()
print("sanitize case ok")
