"""GPU batch-size controller: the reference's DTAHE scheduler (Alg. 3,
PAPER.md:1177-1191) re-targeted at a GPU-only search path.

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
`backend` (launch / poll), so the same code drives the B200 (CudaBackend:
CUDA events, two streams) and the CPU tests (a simulated device).
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


class CudaBackend:
    """Dispatch batches of a device-resident query tensor to a search callable
    on `slots` CUDA streams; completion times come from CUDA events relative to
    a start event, on the same clock as the controller (seconds since start)."""

    def __init__(self, search_fn, queries, k: int, slots: int = 2, max_batch: int = 8192):
        import torch
        self.torch = torch
        self.search_fn = search_fn      # search_fn(queries_slice, out, stream)
        self.queries = queries
        dev = queries.device
        # One stream for all slots: a slot bounds the batches outstanding, the
        # batches themselves run back to back (measured: two streams whose
        # kernels overlap lose ~10 % to interference).
        stream = torch.cuda.Stream(device=dev)
        self.streams = [stream] * slots
        self.outs = [(torch.empty((max_batch, k), dtype=torch.uint64, device=dev),
                      torch.empty((max_batch, k), dtype=torch.uint32, device=dev),
                      torch.empty((max_batch,), dtype=torch.uint32, device=dev)) for _ in range(slots)]
        self.clock = None
        self.start = None

    def begin(self):
        """Synchronise and pin t=0 of both clocks; returns the host clock."""
        torch = self.torch
        torch.cuda.synchronize()
        self.start = torch.cuda.Event(enable_timing=True)
        self.start.record(self.streams[0])
        self.start.synchronize()
        self.clock = _WallClock()
        return self.clock

    def launch(self, first: int, count: int, slot: int):
        torch = self.torch
        st = self.streams[slot]
        out = tuple(o[:count] for o in self.outs[slot])
        with torch.cuda.stream(st):
            self.search_fn(self.queries[first:first + count], out, st)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(st)
        return ev

    def poll(self, ev):
        if not ev.query():
            return None
        return self.start.elapsed_time(ev) * 1e-3


def spin_idle(clock):
    def idle(t_next):
        # short spin: batches finish in ~0.1-10 ms
        if t_next == np.inf:
            time.sleep(20e-6)
            return
        d = t_next - clock()
        if d > 200e-6:
            time.sleep(min(d, 1e-3) - 100e-6)
    return idle


class ShardedBackend:
    """Multi-GPU serving (configs[4]): rank 0 runs the controller; every
    dispatch sends (first, count) to the other ranks over a host-side (gloo)
    group, and all ranks enqueue the sharded search of that batch, whose NCCL
    all-gather keeps the GPUs in lockstep; rank 0 observes completion.  The
    command channel never waits on a GPU, so with `slots` = 2 every rank
    enqueues batch b+1 while batch b runs (double buffering);
    consecutive batches' collectives are issued in the same order on every
    rank, which keeps them matched."""

    STOP = -1

    def __init__(self, search_fn, queries, k: int, max_batch: int = 8192, slots: int = 2, cmd_group=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.search_fn = search_fn  # search_fn(queries_slice, out)
        self.queries = queries
        dev = queries.device
        self.group = cmd_group if cmd_group is not None else dist.new_group(backend="gloo")
        self.cmd = torch.zeros(2, dtype=torch.int64)  # host tensor: gloo
        self.outs = [(torch.empty((max_batch, k), dtype=torch.uint64, device=dev),
                      torch.empty((max_batch, k), dtype=torch.uint32, device=dev),
                      torch.empty((max_batch,), dtype=torch.uint32, device=dev)) for _ in range(slots)]
        self.start = None
        self.clock = None

    def _run_batch(self, first: int, count: int, slot: int):
        out = tuple(o[:count] for o in self.outs[slot])
        self.search_fn(self.queries[first:first + count], out)

    def begin(self):
        torch = self.torch
        torch.cuda.synchronize()
        self.start = torch.cuda.Event(enable_timing=True)
        self.start.record()
        self.start.synchronize()
        self.clock = _WallClock()
        return self.clock

    def _send(self, first: int, count: int, slot: int):
        import torch.distributed as dist
        self.cmd[0], self.cmd[1] = first, (count << 8) | slot
        dist.broadcast(self.cmd, 0, group=self.group)

    def launch(self, first: int, count: int, slot: int):
        self._send(first, count, slot)
        self._run_batch(first, count, slot)
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def poll(self, ev):
        if not ev.query():
            return None
        return self.start.elapsed_time(ev) * 1e-3

    def stop(self):
        self._send(self.STOP, 0, 0)

    def follow(self):
        """Non-zero ranks: run every broadcast batch until the stop command."""
        import torch.distributed as dist
        gc_on = gc.isenabled()
        gc.disable()
        try:
            self._follow(dist)
        finally:
            if gc_on:
                gc.enable()

    def _follow(self, dist):
        while True:
            dist.broadcast(self.cmd, 0, group=self.group)
            first, word = int(self.cmd[0]), int(self.cmd[1])
            if first == self.STOP:
                break
            self._run_batch(first, word >> 8, word & 0xFF)
