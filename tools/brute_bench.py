"""(A/B switches: run against a knob build, HCG_LIB_OVERRIDE=$(python tools/build_variant.py knobs).)
K5 ground-truth throughput: tensor-core (tcgen05 kind::i8) vs CUDA-core
brute force, 10M lifted rows x 1000 queries, k=10.  Run twice, once with
HCG_BRUTE_CUDA_CORES=1 (the env var is read once per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, nq, k = int(os.environ.get("N", 10_000_000)), int(os.environ.get("NQ", 1000)), 10
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = H.gen_queries(0, nq, n)
ids, sq, ln = ix.brute_force(qs, k)  # warm-up
times = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    ids2, sq2, ln2 = ix.brute_force(qs, k)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
ms = sorted(times)[2]
macs = float(n) * nq * 128
print(json.dumps({"path": "cuda_cores" if os.environ.get("HCG_BRUTE_CUDA_CORES") else "tcgen05", "n": n, "nq": nq,
                  "k": k, "ms": ms, "tera_int8_ops_per_s": 2 * macs / (ms * 1e-3) / 1e12,
                  "row_GB_per_s": n * 128 / (ms * 1e-3) / 1e9,
                  "ids_checksum": int(ids2.to(torch.int64).sum().item())}), flush=True)
