"""The GPU batch-size controller (libhcg hcg_server_*, csrc/serve.cpp): the
reference's DTAHE buffer dispatch (Alg. 3)
with the CPU branch removed, run by a C++ dispatcher over one index or one
shard group.  Response times include the queries' H2D and the results' D2H.

    srv = Server(index_or_group, k=10, depth=350)          # policy defaults: B=8192, 2 in flight
    ids, sq, ln, lat, sizes = srv.replay(queries_u8, arrivals_s)   # open-loop trace
    srv.start(capacity=1 << 16); t = srv.submit(q); ids, sq, ln, lat = srv.wait(t)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import HcgServerPolicy, check, lib


class Server:
    def __init__(self, target, k: int, depth: int, max_batch: int = 8192, min_batch: int = 1,
                 max_wait: float = 0.0, slots: int = 2):
        from .sharded import ShardGroup
        self.k = k
        self.target = target  # keeps the index / group alive
        pol = HcgServerPolicy(max_batch, min_batch, max_wait, slots)
        h = C.c_void_p()
        if isinstance(target, ShardGroup):
            check(lib().hcg_server_create(None, target._h, k, depth, C.byref(pol), C.byref(h)))
            self.d_full = target.d_full
        else:
            check(lib().hcg_server_create(target._h, None, k, depth, C.byref(pol), C.byref(h)))
            self.d_full = target.scheme.d_full
        self._h = h
        self.max_batch = max_batch

    def replay(self, queries, arrivals):
        """Open-loop replay of host queries arriving at `arrivals` (seconds,
        non-decreasing).  Returns ids, sqdist, len, latency (s), batch sizes."""
        q = np.ascontiguousarray(queries, np.uint8)
        arr = np.ascontiguousarray(arrivals, np.float64)
        nq = q.shape[0]
        assert arr.shape[0] == nq and q.shape[1] == self.d_full
        ids = np.empty((nq, self.k), np.uint64)
        sq = np.empty((nq, self.k), np.uint32)
        ln = np.empty(nq, np.uint32)
        lat = np.empty(nq, np.float64)
        sizes = np.empty(max(nq, 1), np.uint32)
        nb = C.c_uint32()
        check(lib().hcg_server_replay(self._h, q.ctypes.data, nq, arr.ctypes.data, ids.ctypes.data, sq.ctypes.data,
                                      ln.ctypes.data, lat.ctypes.data, sizes.ctypes.data, C.byref(nb)))
        return ids, sq, ln, lat, sizes[:nb.value].copy()

    def start(self, capacity: int = 1 << 16) -> None:
        check(lib().hcg_server_start(self._h, capacity))

    def submit(self, queries) -> int:
        q = np.ascontiguousarray(queries, np.uint8).reshape(-1, self.d_full)
        t = C.c_uint64()
        check(lib().hcg_server_submit(self._h, q.ctypes.data, q.shape[0], C.byref(t)))
        self._pending = getattr(self, "_pending", {})
        self._pending[t.value] = q.shape[0]
        return t.value

    def wait(self, ticket: int):
        nq = self._pending.pop(ticket)
        ids = np.empty((nq, self.k), np.uint64)
        sq = np.empty((nq, self.k), np.uint32)
        ln = np.empty(nq, np.uint32)
        lat = np.empty(nq, np.float64)
        check(lib().hcg_server_wait(self._h, ticket, ids.ctypes.data, sq.ctypes.data, ln.ctypes.data,
                                    lat.ctypes.data))
        return ids, sq, ln, lat

    def close(self) -> None:
        if self._h:
            lib().hcg_server_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def latency_summary(lat_s: np.ndarray, sizes: np.ndarray, makespan_s: float | None = None) -> dict:
    lat = np.asarray(lat_s) * 1e3
    bs = np.asarray(sizes)
    out = {"queries": int(len(lat)),
           "latency_ms": {"mean": float(lat.mean()), "p50": float(np.percentile(lat, 50)),
                          "p99": float(np.percentile(lat, 99)), "max": float(lat.max())},
           "batches": int(len(bs)),
           "batch_size": {"mean": float(bs.mean()), "p50": float(np.percentile(bs, 50)), "max": int(bs.max())}}
    if makespan_s:
        out["throughput_qps"] = float(len(lat) / makespan_s)
    return out
