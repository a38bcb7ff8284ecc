"""Batch-size controller (DTAHE, Alg. 3 without its CPU branch) on a
simulated device with a virtual clock: SPEC.md acceptance 5's properties that
survive the GPU-only re-targeting -- task conservation (5d), small batches
under light load (5b), full batches under saturation (5c), FIFO service."""
import numpy as np
import pytest

from paper_1209_0410_b200.controller import BatchController, Policy, poisson_arrivals


class SimDevice:
    """One batch at a time (FIFO), service = fixed + per-query cost (seconds)."""

    def __init__(self, fixed=100e-6, per_query=0.1e-6):
        self.fixed, self.per_query = fixed, per_query
        self.busy_until = 0.0
        self.clock = None
        self.log = []

    def launch(self, first, count, slot):
        start = max(self.clock.t, self.busy_until)
        self.busy_until = start + self.fixed + self.per_query * count
        self.log.append((first, count, slot, start, self.busy_until))
        return self.busy_until

    def poll(self, token):
        return token if token <= self.clock.t + 1e-15 else None


class VClock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t


def run(arrivals, policy):
    dev = SimDevice()
    clk = VClock()
    dev.clock = clk
    def idle(t_next):
        nxt_done = min([e[4] for e in dev.log if e[4] > clk.t], default=np.inf)
        clk.t = max(clk.t, min(t_next, nxt_done))
    res = BatchController(policy).run(arrivals, dev, clock=clk, idle=idle)
    return res, dev


def test_conservation_fifo_and_bounds():
    arr = poisson_arrivals(2e6, 20000, seed=1)
    res, dev = run(arr, Policy(max_batch=512))
    assert len(res.latency) == 20000 and (res.latency >= 0).all()
    firsts = [e[0] for e in dev.log]
    counts = [e[1] for e in dev.log]
    assert firsts == sorted(firsts)
    assert sum(counts) == 20000 and max(counts) <= 512
    assert all(firsts[i] + counts[i] == firsts[i + 1] for i in range(len(firsts) - 1))  # contiguous, FIFO


def test_light_load_gives_small_batches():
    # device can do ~1/(100us) batches/s; arrivals every ~1ms -> one query per batch
    arr = poisson_arrivals(1e3, 2000, seed=2)
    res, _ = run(arr, Policy())
    assert np.mean(res.batch_sizes) < 1.2
    assert np.percentile(res.latency, 50) < 150e-6


def test_saturation_fills_batches():
    arr = np.zeros(200000)
    res, _ = run(arr, Policy(max_batch=8192))
    full = np.mean(np.asarray(res.batch_sizes) == 8192)
    assert full >= 0.9
    # throughput close to the device's batched capacity (fixed cost amortised)
    cap = 8192 / (100e-6 + 0.1e-6 * 8192)
    assert res.summary()["throughput_qps"] >= 0.9 * cap


def test_latency_grows_with_load():
    p50 = []
    for rate in (1e5, 1e6, 5e6, 8e6):
        res, _ = run(poisson_arrivals(rate, 30000, seed=3), Policy(max_batch=8192))
        p50.append(np.percentile(res.latency, 50))
    assert p50 == sorted(p50)


def test_min_batch_and_max_wait_trade_latency_for_batching():
    arr = poisson_arrivals(2e5, 20000, seed=4)
    eager, _ = run(arr, Policy(max_batch=8192))
    held, _ = run(arr, Policy(max_batch=8192, min_batch=64, max_wait=200e-6))
    assert np.mean(held.batch_sizes) > np.mean(eager.batch_sizes)
    # (with a 100 us fixed cost per batch, holding queries back can even LOWER the
    # median latency -- the queueing effect DTAHE exploits; only bound it here)
    assert held.latency.max() <= 200e-6 + 100e-6 + 0.1e-6 * 8192 + 200e-6
