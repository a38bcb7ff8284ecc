"""Sharded search over one process per GPU (the reference's hypershard module,
SPEC.md:338-419).

partition : global id i lives on rank i mod G at local slot i // G
             -- the index is built with id_base=r, id_stride=G,
            so every result already carries its global id.
broadcast : every rank receives the same query batch.
IHLS      : each rank searches its shard at the per-shard probe depth
            (plan_depth for a miss-probability target).
aggregate : one NCCL all-gather of the packed (sqdist<<32 | gid) top-k lists
            (B x k x 8 bytes per rank), then the K4 merge kernel by
            (distance, id), truncated to k.  The exchange is
            the only device-to-device traffic of the path.

The search runs inside libhcg (hcg_shard_group_*, csrc/shard.cu): the
library owns the NCCL communicators and issues the all-gather itself;
torch.distributed only carries the NCCL id at join time and the recall /
parity side computations outside the timed path.
"""
from __future__ import annotations

import numpy as np

import ctypes as C

from ._lib import HcgNcclId, check, lib
from .multicurves import (MulticurvesIndex, ProjectionScheme, View, _empty_like_kind, _ptr, _stream, _u8_2d,
                          c_scheme, gen_rows, merge_packed)


def shard_rows(n_total: int, rank: int, world: int) -> int:
    """Number of global ids i < n_total with i mod world == rank."""
    return 0 if rank >= n_total else (n_total - rank + world - 1) // world


def exchange(packed, world: int, group=None, out=None):
    """The aggregate's only collective: all-gather every rank's packed
    (sqdist << 32 | gid) top-k block [nq, k] into [world, nq, k] (NCCL over
    NVLink on GPUs; any torch.distributed backend works)."""
    import torch
    import torch.distributed as dist
    nq, k = int(packed.shape[0]), int(packed.shape[1])
    if out is None:
        out = torch.empty((world, nq, k), dtype=packed.dtype, device=packed.device)
    src = packed.contiguous()
    if src.dtype == torch.uint64:  # NCCL/gloo move 64-bit payloads as int64
        src = src.view(torch.int64)
        dst = out.view(torch.int64)
    else:
        dst = out
    dist.all_gather_into_tensor(dst.view(-1), src.view(-1), group=group)
    return out


def pack(ids, sqdist, lens, k: int):
    """Packed (sqdist << 32 | id) per result, -1 (all ones) past each list's length."""
    import torch
    p = (sqdist.to(torch.int64) << 32) | ids.view(torch.int64)
    valid = lens.view(-1, 1).to(torch.int64) > torch.arange(k, device=ids.device)
    return torch.where(valid, p, torch.full_like(p, -1))


class ShardGroup:
    """hcg_shard_group (include/hcg.h): the partition / aggregate inside
    libhcg -- per-shard search, ncclAllGather of the packed top-k lists over
    NVLink and the K4 merge, driven from C++.  No torch.distributed on the
    search path; torch.distributed only hands the NCCL id to the ranks once
    (join)."""

    def __init__(self, handle, d_full: int, keep=()):
        self._h = handle
        self.d_full = d_full
        self._keep = list(keep)

    @classmethod
    def build(cls, rows, scheme: ProjectionScheme, view: View, devices) -> "ShardGroup":
        """One process, G = len(devices) GPUs: shard r (rows r, r+G, ...) on devices[r]."""
        r = _u8_2d(rows, scheme.d_full)
        s = c_scheme(scheme, view)
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        check(lib().hcg_shard_group_build(C.byref(s), _ptr(r), r.shape[0], len(devices), devs, C.byref(h)))
        return cls(h, scheme.d_full)

    @classmethod
    def adopt(cls, shards) -> "ShardGroup":
        """One process over already-built shards (shard r: id_base r, id_stride G,
        one per GPU); the group takes them over (the Python objects are emptied)."""
        G = len(shards)
        arr = (C.c_void_p * G)(*[x._h.value if isinstance(x._h, C.c_void_p) else x._h for x in shards])
        h = C.c_void_p()
        check(lib().hcg_shard_group_adopt(G, arr, C.byref(h)))
        for x in shards:
            x._h = None
        return cls(h, shards[0].scheme.d_full)

    @classmethod
    def join(cls, local: MulticurvesIndex, rank: int, world: int, pg=None) -> "ShardGroup":
        """One process per GPU (collective): rank 0 makes the NCCL id, the
        process group carries it to every rank, each joins with its shard."""
        import torch
        import torch.distributed as dist
        nid = HcgNcclId()
        if rank == 0:
            check(lib().hcg_nccl_unique_id(C.byref(nid)))
        backend = dist.get_backend(pg)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        t = torch.tensor(list(bytes(nid.internal)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0, group=pg)
        C.memmove(C.addressof(nid), bytes(t.cpu().tolist()), 128)
        h = C.c_void_p()
        check(lib().hcg_shard_group_join(C.byref(nid), rank, world, local._h, C.byref(h)))
        return cls(h, local.scheme.d_full, keep=[local])

    def shards(self) -> int:
        return int(lib().hcg_shard_group_shards(self._h))

    def search(self, queries, k: int, shard_depth: int, out=None, stream=None):
        """Global top-k (ids u64, sqdist u32, len u32) of a query batch."""
        q = _u8_2d(queries, self.d_full)
        nq = q.shape[0]
        if out is None:
            ids = _empty_like_kind(q, (nq, k), np.uint64)
            sq = _empty_like_kind(q, (nq, k), np.uint32)
            ln = _empty_like_kind(q, (nq,), np.uint32)
        else:
            ids, sq, ln = out
        check(lib().hcg_shard_group_search(self._h, _ptr(q), nq, k, shard_depth, _ptr(ids), _ptr(sq), _ptr(ln),
                                           _stream(stream, q)))
        return ids, sq, ln

    def search_routed(self, queries, k: int, shard_depth: int, out=None, stream=None):
        """The aggregate routed to one aggregator per query:
        this rank merges only its query block [first, first + count) of the
        batch and fills those rows of `out`.  Returns (out, first, count)."""
        q = _u8_2d(queries, self.d_full)
        nq = q.shape[0]
        if out is None:
            out = (_empty_like_kind(q, (nq, k), np.uint64), _empty_like_kind(q, (nq, k), np.uint32),
                   _empty_like_kind(q, (nq,), np.uint32))
        ids, sq, ln = out
        first, count = C.c_uint32(), C.c_uint32()
        check(lib().hcg_shard_group_search_routed(self._h, _ptr(q), nq, k, shard_depth, _ptr(ids), _ptr(sq), _ptr(ln),
                                                  _stream(stream, q), C.byref(first), C.byref(count)))
        return out, first.value, count.value

    def close(self) -> None:
        if self._h:
            lib().hcg_shard_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedIndex:
    """One rank's share of a G-way sharded Multicurves index."""

    def __init__(self, local: MulticurvesIndex, rank: int, world: int, group=None):
        self.local = local
        self.rank = rank
        self.world = world
        self.group = group
        self._bufs = {}
        # the search path: libhcg's shard group (NCCL inside the library)
        self.shard_group = ShardGroup.join(local, rank, world, group) if world > 1 else None

    @classmethod
    def from_generator(cls, n_total: int, scheme: ProjectionScheme, view: View, rank: int, world: int,
                       device: int, group=None) -> "ShardedIndex":
        """Each rank generates exactly its own rows (i = rank + s*world) on its GPU."""
        cnt = shard_rows(n_total, rank, world)
        rows = gen_rows(rank, cnt, stride=world, device=device)
        local = MulticurvesIndex(rows, scheme, view, device=device, id_base=rank, id_stride=world)
        del rows
        return cls(local, rank, world, group)

    def _buf(self, key, shape, dtype, device):
        """A view of a grow-only scratch buffer: batches of varying size (the
        online controller) reuse one allocation instead of the allocator."""
        import torch
        numel = 1
        for x in shape:
            numel *= int(x)
        b = self._bufs.get(key)
        if b is None or b.numel() < numel:
            b = torch.empty(max(numel, 1), dtype=dtype, device=device)
            self._bufs[key] = b
        return b[:numel].view(shape)

    def search(self, queries, k: int, shard_depth: int, out=None):
        """Global top-k of a query batch (device tensors in and out).

        queries: [nq, d] uint8 CUDA tensor (the broadcast batch, same on every rank).
        Returns (ids u64, sqdist u32, len u32) CUDA tensors, identical on all ranks.
        """
        if self.world == 1:
            return self.local.search_batch(queries, k, shard_depth, out=out)
        return self.shard_group.search(queries, k, shard_depth, out=out)

    def search_torch(self, queries, k: int, shard_depth: int, out=None):
        """The same aggregate through torch.distributed (packed search, all-gather
        of the packed lists, K4): the pre-shard-group path, kept to cross-check."""
        import torch
        dev = queries.device
        nq = int(queries.shape[0])
        packed = self._buf("packed", (nq, k), torch.uint64, dev)
        self.local.search_packed(queries, k, shard_depth, out=packed)
        gathered = self._buf("gathered", (self.world, nq, k), torch.uint64, dev)
        exchange(packed, self.world, self.group, out=gathered)
        return merge_packed(gathered, k, device=dev.index, out=out)

    def brute_force(self, queries, k: int):
        """Exact global top-k (recall ground truth): per-shard exact lists merged the same way."""
        import torch
        ids, sq, ln = self.local.brute_force(queries, k)
        if self.world == 1:
            return ids, sq, ln
        gathered = exchange(pack(ids, sq, ln, k), self.world, self.group)
        return merge_packed(gathered.view(torch.uint64), k, device=ids.device.index)


def recall(found_ids, true_ids, k: int) -> float:
    f = np.asarray(found_ids)[:, :k]
    t = np.asarray(true_ids)[:, :k]
    none = np.uint64(2**64 - 1)
    hits = sum(len((set(a.tolist()) & set(b.tolist())) - {int(none)}) for a, b in zip(f, t))
    return hits / float(k * max(len(f), 1))
