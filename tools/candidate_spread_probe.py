"""How concentrated are a query's candidate rows in the physical (curve-0)
order?  Fraction of each query's unique candidates within a window of W rows
around the median physical position (a bitmap union over such a window
would dedup those ids without hashing)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n = 10_000_000
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
order0 = ix.subindex(0).astype(np.int64)        # ids in curve-0 order = physical order
phys = np.empty(n, np.int64)
phys[order0] = np.arange(n)
qs = H.gen_queries(0, 200, n).cpu().numpy()
cands = ix.candidates(qs, 350)
for W in (1 << 14, 1 << 16, 1 << 18, 1 << 20):
    fr = []
    for c in cands:
        p = np.sort(phys[c.astype(np.int64)])
        # best window of W rows (max count) via two pointers
        j = 0
        best = 0
        for i in range(len(p)):
            while p[i] - p[j] >= W:
                j += 1
            best = max(best, i - j + 1)
        fr.append(best / len(p))
    print(f"window {W:8d} rows: best-window share of candidates mean {np.mean(fr):.3f} p10 {np.percentile(fr, 10):.3f}",
          flush=True)
