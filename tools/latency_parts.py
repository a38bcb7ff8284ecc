"""Per-kernel device time of small batches (locate / union / gather) plus the
host-observed latency of one search call."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n = 10_000_000
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = H.gen_queries(0, 4096, n)
for bs in (1, 16, 256, 4096):
    q = qs[:bs].contiguous()
    out = (torch.empty((bs, 10), dtype=torch.uint64, device="cuda"), torch.empty((bs, 10), dtype=torch.uint32, device="cuda"),
           torch.empty((bs,), dtype=torch.uint32, device="cuda"))
    for _ in range(5):
        ix.search_batch(q, 10, 350, out=out)
    parts = [ix.search_timed(q, 10, 350, out=out) for _ in range(20)]
    med = [sorted(p[i] for p in parts)[10] for i in range(3)]
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        ix.search_batch(q, 10, 350, out=out)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"batch={bs:5d} locate={med[0]*1e3:7.1f}us union={med[1]*1e3:7.1f}us gather={med[2]*1e3:7.1f}us "
          f"host_p50={ts[25]*1e6:7.1f}us", flush=True)
