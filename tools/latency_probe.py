"""Where the small-batch latency goes (10M lifted, k=10, depth 350, one B200):
per batch size, the host time of one hcg_search call from Python (no sync),
the same from C (the call alone, timed by ctypes around it), and the device
span of the call (CUDA events around it, as bench.py's latency).  Kernel
durations come from the ncu launch list of the same run."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n = int(os.environ.get("PROBE_N", 10_000_000))
ix = H.MulticurvesIndex(H.gen_rows(0, n), H.default_scheme(128, 8, 16), H.LIFTED)
qs = H.gen_queries(0, 4096, n)
L = H.lib()
st = torch.cuda.current_stream()
for bs in (1, 16, 64, 128, 256, 512):
    q = qs[:bs].contiguous()
    out = (torch.empty((bs, 10), dtype=torch.uint64, device="cuda"), torch.empty((bs, 10), dtype=torch.uint32, device="cuda"),
           torch.empty((bs,), dtype=torch.uint32, device="cuda"))
    args = (ix._h, q.data_ptr(), bs, 10, 350, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), st.cuda_stream)
    for _ in range(10):
        ix.search_batch(q, 10, 350, out=out)
    torch.cuda.synchronize()
    # host: python wrapper, then raw ctypes (no Python-side argument handling)
    t0 = time.perf_counter()
    for _ in range(200):
        ix.search_batch(q, 10, 350, out=out)
    t_py = (time.perf_counter() - t0) / 200
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        L.hcg_search(*args)
    t_c = (time.perf_counter() - t0) / 200
    torch.cuda.synchronize()
    dev = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.hcg_search(*args)
        e1.record(st)
        e1.synchronize()
        dev.append(e0.elapsed_time(e1))
    # back-to-back device throughput of the kernel chain (host runs ahead)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(100):
        L.hcg_search(*args)
    e1.record(st)
    e1.synchronize()
    print(json.dumps({"batch": bs, "host_us_python_call": round(t_py * 1e6, 1), "host_us_c_call": round(t_c * 1e6, 1),
                      "device_span_us_p50": round(float(np.median(dev)) * 1e3, 1),
                      "device_us_per_call_back_to_back": round(e0.elapsed_time(e1) * 1e3 / 100, 1)}), flush=True)
