"""Float-descriptor (HCG_F32) search at the bench scale: 10M x 128 f32 rows =
the generator's bytes in the lifted view (1 + b/256, exact in f32), 100K
queries, k=10, depth 350, 8 curves, m=16.

Because the lifted floats are exact, every f32 squared distance equals the
u8 index's integer sqdist / 65536 exactly: the f32 index must return the
same ids as the u8 lifted index -- a full-scale cross-check of the f32
kernels.  Prints one JSON line (q/s, ms/step, gather bandwidth)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n = int(os.environ.get("F32_N", 10_000_000))
nq, k, depth = 100_000, 10, 350
scheme = H.default_scheme(128, 8, 16)
rows8 = H.gen_rows(0, n)
ix8 = H.MulticurvesIndex(rows8, scheme, H.LIFTED)
rowsf = 1.0 + rows8.to(torch.float32) / 256.0
del rows8
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
ixf = H.MulticurvesIndex(rowsf, scheme)
t1.record()
torch.cuda.synchronize()
build_ms = t0.elapsed_time(t1)
del rowsf
q8 = H.gen_queries(0, nq, n)
qf = 1.0 + q8.to(torch.float32) / 256.0

ids8, sq8, ln8 = ix8.search_batch(q8, k, depth)
idsf, sqf, lnf = ixf.search_batch(qf, k, depth)
torch.cuda.synchronize()
same_ids = bool(torch.equal(ids8, idsf) and torch.equal(ln8, lnf))
same_dist = bool(torch.equal(sq8.to(torch.float64) / 65536.0, sqf))
U = int(ix8.candidate_counts(q8[:2000].cpu().numpy(), depth).astype("int64").sum()) * nq / 2000

out = (idsf, sqf, lnf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
times = []
for it in range(8):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ixf.search_batch(qf, k, depth, out=out)
    b.record()
    torch.cuda.synchronize()
    if it >= 3:
        times.append(a.elapsed_time(b))
ms = sorted(times)[len(times) // 2]
print(json.dumps({
    "workload": f"f32 lifted {n} x 128, {nq} queries, k={k}, depth={depth}, 8 curves, m=16",
    "queries_per_s": nq / (ms * 1e-3), "ms_per_step": ms, "build_ms": build_ms,
    "unique_candidates_per_query": U / nq,
    "gathered_GB_per_s_lower_bound": U * 512 / (ms * 1e-3) / 1e9,
    "ids_equal_u8_index": same_ids, "dist_equal_u8_index": same_dist,
}))
