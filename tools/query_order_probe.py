"""(A/B switches: run against a knob build, HCG_LIB_OVERRIDE=$(python tools/build_variant.py knobs).)
Probe: which batch order gives the gather the most L2 reuse?  Times
search_timed (batch-order sort disabled, HCG_NO_QSORT=1) on the same queries
pre-sorted on the host by: generator order, curve-0 rank, a coarse Z-order key
over many dimensions (top bits of 32 / 64 dims interleaved)."""
import os
import sys

import numpy as np
import torch

os.environ["HCG_NO_QSORT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D = 10_000_000, 100_000, 10, 350
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = [H.gen_queries(b * Q, Q, n) for b in range(2)]


def zkey(qh, dims, bits):
    """Interleave the top `bits` bits of `dims` dims (first bit plane most significant)."""
    key = np.zeros(qh.shape[0], dtype=object)
    parts = []
    for b in range(bits):
        for d in dims:
            parts.append((qh[:, d] >> (7 - b)) & 1)
    # pack into python ints via numpy bytes
    arr = np.stack(parts, axis=1).astype(np.uint8)
    packed = np.packbits(arr, axis=1)
    return [bytes(r) for r in packed]


orders = {}
for b, q in enumerate(qs):
    qh = q.cpu().numpy()
    r, _, _ = ix.windows(qh, D)
    orders.setdefault("generator", []).append(np.arange(Q))
    orders.setdefault("curve0_rank", []).append(np.argsort(r[:, 0], kind="stable"))
    for nd, bits in ((32, 2), (64, 1), (128, 1)):
        kk = zkey(qh, list(range(0, 128, 128 // nd)), bits)
        orders.setdefault(f"zorder_{nd}dims_{bits}bits", []).append(np.array(sorted(range(Q), key=kk.__getitem__)))
    # curve ranks lexicographic over coarse buckets of curves 0..3
    coarse = (r[:, :4] >> 12).astype(np.int64)
    orders.setdefault("coarse4curves", []).append(np.lexsort(coarse.T[::-1]))
out = (torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
       torch.empty((Q,), dtype=torch.uint32, device="cuda"))
for name, ords in orders.items():
    batches = [qs[b][torch.from_numpy(ords[b].astype(np.int64)).cuda()].contiguous() for b in range(2)]
    for b in range(2):
        ix.search_timed(batches[b], k, D, out=out)
    t = [ix.search_timed(batches[b % 2], k, D, out=out) for b in range(6)]
    med = [sorted(x[i] for x in t)[3] for i in range(3)]
    print(f"{name}: union {med[1]:.3f} gather {med[2]:.3f} ms", flush=True)
