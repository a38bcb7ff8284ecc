"""Phase times of the small-batch kernel (k_search_small) for one query:
run against a tuning build with HCG_SMALL_PROF=1
(HCG_LIB_OVERRIDE=$(python tools/build_variant.py knobs)); the library prints
the locate / union / gather / merge spans (globaltimer) to stderr."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n = 10_000_000
ix = H.MulticurvesIndex(H.gen_rows(0, n), H.default_scheme(128, 8, 16), H.LIFTED)
qs = H.gen_queries(0, 64, n)
for i in range(20):
    ix.search_batch(qs[i:i + 1].contiguous(), 10, 350)
torch.cuda.synchronize()
