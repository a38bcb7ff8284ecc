"""A/B: device-resident search steps on the legacy default stream vs a
created stream (10M lifted, 100K queries, k=10, D=350)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402

n, Q, k, D = 10_000_000, 100_000, 10, 350
rows = H.gen_rows(0, n)
ix = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
del rows
qs = [H.gen_queries(b * Q, Q, n) for b in range(13)]
out = (torch.empty((Q, k), dtype=torch.uint64, device="cuda"), torch.empty((Q, k), dtype=torch.uint32, device="cuda"),
       torch.empty((Q,), dtype=torch.uint32, device="cuda"))


def run(stream):
    with torch.cuda.stream(stream):
        for b in range(3):
            ix.search_batch(qs[b], k, D, out=out)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for b in range(3, 13):
            ix.search_batch(qs[b], k, D, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


s = torch.cuda.Stream()
for name, st in [("default", torch.cuda.default_stream()), ("created", s)] * 3:
    print(f"{name}: {run(st):.3f} ms/step", flush=True)

# the same with an nvidia-smi poller (bench.py's clock sampler) and an
# in-process NVML poller running
import subprocess  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,utilization.gpu", "--format=csv,noheader",
                      "-lms", "100"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
time.sleep(0.5)
for _ in range(3):
    print(f"with nvidia-smi -lms 100: {run(s):.3f} ms/step", flush=True)
p.terminate()
p.wait()
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False


def poll():
    while not stop:
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        pynvml.nvmlDeviceGetUtilizationRates(h)
        time.sleep(0.1)


t = threading.Thread(target=poll, daemon=True)
t.start()
for _ in range(3):
    print(f"with NVML poll 100 ms: {run(s):.3f} ms/step", flush=True)
stop = True
for _ in range(2):
    print(f"no poller: {run(s):.3f} ms/step", flush=True)
