"""(A/B switches: run against a knob build, HCG_LIB_OVERRIDE=$(python tools/build_variant.py knobs).)
Time the refine kernel on the bench workload (10M lifted, 100K queries,
k=10, depth $DEPTH) and print its per-launch device time and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D = 10_000_000, 100_000, int(os.environ.get("K", "10")), int(os.environ.get("DEPTH", "350"))
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = [H.gen_queries(b * Q, Q, n) for b in range(4)]
out = (torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
       torch.empty((Q,), dtype=torch.uint32, device="cuda"))
U = ix.candidate_counts(qs[0], D).astype("float64")
bytes_ = U.sum() * 128 + Q * (4 * 8 * D + 4 * 8 + 128) + Q * (12 * k + 4)
for b in range(2):
    ix.search_timed(qs[b], k, D, out=out)
t = [ix.search_timed(qs[b % 4], k, D, out=out) for b in range(8)]
loc = sorted(x[0] for x in t)[4]
uni = sorted(x[1] for x in t)[4]
gat = sorted(x[2] for x in t)[4]
ref = uni + gat
print(f"depth={D} k={k} U={U.mean():.1f} locate_ms={loc:.3f} union_ms={uni:.3f} gather_ms={gat:.3f} "
      f"refine_ms={ref:.3f} refine_GB/s={bytes_ / ref / 1e6:.0f}", flush=True)



if os.environ.get("UNION_AB"):
    for v in ("reg", "smem", "reg", "smem"):
        if v == "smem":
            os.environ["HCG_UNION_SMEM"] = "1"
        else:
            os.environ.pop("HCG_UNION_SMEM", None)
        for b in range(2):
            ix.search_timed(qs[b], k, D, out=out)
        ms = sorted(ix.search_timed(qs[b % 4], k, D, out=out)[1] for b in range(6))[3]
        print(f"union={v} union_ms={ms:.3f}", flush=True)




