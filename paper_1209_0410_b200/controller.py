"""Simulation model of the GPU batch-size controller: the reference's DTAHE
scheduler (Alg. 3) re-targeted at a
GPU-only search path.  The product controller is C++ (libhcg hcg_server_*,
csrc/serve.cpp, Python handle server.Server); this module states the same
dispatch rule over an abstract backend so that its properties are tested on
CPU against a simulated device (SPEC.md's `simulate` operation: virtual clock,
deterministic), and provides the Poisson workload generator.

DTAHE routes each arriving query either to a CPU core (lines 3-4) or into the
current GPU buffer, and queues the buffer on the device when the device is
idle or the buffer is full (lines 9-10); at most two buffers are alive
(double buffering).  The north star drops the CPU branch (no CPU
fallback), which leaves the buffer rule as a batch-size controller:

  * at most `slots` batches in flight (2 = double buffer);
  * when a slot is free, dispatch min(queue, max_batch) queries at once if the
    device is idle (DTAHE "GPU idle"), or if the queue already holds
    `min_batch` queries (DTAHE "buffer full"), or if the oldest waiting query
    has waited `max_wait` seconds;
  * otherwise keep buffering.

Batch size therefore follows the load: ~1 query per batch when lightly loaded
(latency = one search), growing towards max_batch near saturation (throughput
= the batched kernels').  Queries are served FIFO, so each batch is a
contiguous range of the arrival sequence.

The policy is independent of time and device: `run()` takes a `clock` and a
`backend` (launch / poll).
"""
from __future__ import annotations

import gc
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Policy:
    max_batch: int = 8192
    min_batch: int = 1
    max_wait: float = 0.0  # seconds; 0 = never hold a query back when a slot is free
    slots: int = 2


@dataclass
class RunResult:
    latency: np.ndarray          # seconds per query (completion - arrival)
    completion: np.ndarray       # seconds since start
    batch_sizes: list = field(default_factory=list)
    batch_starts: list = field(default_factory=list)
    makespan: float = 0.0

    def summary(self) -> dict:
        lat = self.latency * 1e3
        bs = np.asarray(self.batch_sizes)
        return {
            "queries": int(len(lat)),
            "throughput_qps": float(len(lat) / self.makespan) if self.makespan > 0 else None,
            "latency_ms": {"mean": float(lat.mean()), "p50": float(np.percentile(lat, 50)),
                           "p99": float(np.percentile(lat, 99)), "max": float(lat.max())},
            "batches": int(len(bs)),
            "batch_size": {"mean": float(bs.mean()), "p50": float(np.percentile(bs, 50)),
                           "max": int(bs.max())},
        }


class BatchController:
    def __init__(self, policy: Policy | None = None):
        self.policy = policy or Policy()

    def run(self, arrivals: np.ndarray, backend, clock=None, idle=None) -> RunResult:
        """Serve queries with the given arrival times (seconds, non-decreasing).

        backend.launch(first, count, slot) -> token   (start a batch)
        backend.poll(token) -> completion time or None
        clock() -> now; idle(next_event_time) -> None (sleep/spin or advance a
        virtual clock)."""
        gc_on = gc.isenabled()
        gc.disable()  # a full collection mid-run stalls dispatch for milliseconds
        try:
            return self._run(arrivals, backend, clock, idle)
        finally:
            if gc_on:
                gc.enable()

    def _run(self, arrivals, backend, clock, idle) -> RunResult:
        p = self.policy
        arrivals = np.asarray(arrivals, dtype=np.float64)
        n = len(arrivals)
        clock = clock or _WallClock()
        idle = idle or (lambda _t: None)
        completion = np.full(n, np.nan)
        queue_head = 0           # first query not yet dispatched
        arrived = 0              # queries with arrival <= now
        inflight = deque()       # (token, first, count, slot)
        free_slots = list(range(p.slots))
        sizes, starts = [], []
        done = 0
        while done < n:
            now = clock()
            if arrived < n and arrivals[arrived] <= now:  # vectorised: a burst can hold the whole run
                arrived = int(np.searchsorted(arrivals, now, side="right"))
            # retire finished batches (FIFO per slot, any order across slots)
            for item in list(inflight):
                t = backend.poll(item[0])
                if t is not None:
                    completion[item[1]:item[1] + item[2]] = t
                    done += item[2]
                    free_slots.append(item[3])
                    inflight.remove(item)
            waiting = arrived - queue_head
            if free_slots and waiting > 0:
                device_idle = not inflight
                oldest_wait = now - arrivals[queue_head]
                if device_idle or waiting >= p.min_batch or oldest_wait >= p.max_wait:
                    count = min(waiting, p.max_batch)
                    slot = free_slots.pop(0)
                    token = backend.launch(queue_head, count, slot)
                    inflight.append((token, queue_head, count, slot))
                    sizes.append(count)
                    starts.append(now)
                    queue_head += count
                    continue
            # nothing to do right now: wait for the next arrival or completion
            nxt = arrivals[arrived] if arrived < n else np.inf
            if waiting > 0 and free_slots and p.max_wait > 0:
                nxt = min(nxt, arrivals[queue_head] + p.max_wait)
            idle(nxt)
        makespan = float(np.nanmax(completion) - arrivals[0]) if n else 0.0
        assert not np.isnan(completion).any(), "a query was never answered"
        return RunResult(completion - arrivals, completion, sizes, starts, makespan)


def poisson_arrivals(rate: float, n: int, seed: int = 0) -> np.ndarray:
    """exponential inter-arrival times, deterministic under seed."""
    rng = np.random.default_rng(seed)
    return np.cumsum(rng.exponential(1.0 / rate, size=n))


class _WallClock:
    def __init__(self):
        self.t0 = time.perf_counter()

    def __call__(self):
        return time.perf_counter() - self.t0
