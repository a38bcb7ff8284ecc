"""Host-side cost of one search call (enqueue only, device buffers) and the
synchronous latency, for small batches."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, k, D = 10_000_000, 10, 350
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = H.gen_queries(0, 4096, n)
for B in (1, 16, 256):
    q = qs[:B].contiguous()
    out = (torch.empty((B, k), dtype=torch.uint64, device="cuda"), torch.empty((B, k), dtype=torch.uint32, device="cuda"),
           torch.empty((B,), dtype=torch.uint32, device="cuda"))
    for _ in range(20):
        ix.search_batch(q, k, D, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        ix.search_batch(q, k, D, out=out)
    t_enq = (time.perf_counter() - t0) / 200
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) / 200
    lat = []
    for _ in range(200):
        t1 = time.perf_counter()
        ix.search_batch(q, k, D, out=out)
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - t1)
    lat.sort()
    print(f"B={B}: host enqueue {t_enq * 1e6:.1f} us/call, pipelined {t_all * 1e6:.1f} us/call, "
          f"sync latency p50 {lat[100] * 1e6:.1f} us", flush=True)
