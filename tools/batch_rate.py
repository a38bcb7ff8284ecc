"""Throughput of back-to-back batches of a fixed size on one / two streams
(no controller): the ceiling the online controller works against."""
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
qs = H.gen_queries(0, 100_000, n)
for B in (1024, 4096, 8192, 16384):
    outs = [(torch.empty((B, k), dtype=torch.uint64, device="cuda"), torch.empty((B, k), dtype=torch.uint32, device="cuda"),
             torch.empty((B,), dtype=torch.uint32, device="cuda")) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    nb = 100_000 // B
    for ns in (1, 2):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for b in range(nb):
                st = streams[b % ns]
                with torch.cuda.stream(st):
                    ix.search_batch(qs[b * B:(b + 1) * B], k, D, out=outs[b % 2], stream=st)
            t_host = time.perf_counter() - t0
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
        print(f"B={B:6d} streams={ns}: {nb * B / t / 1e6:6.2f} M q/s  ({t / nb * 1e3:.3f} ms/batch, host enqueue "
              f"{t_host / nb * 1e3:.3f} ms/batch)", flush=True)
