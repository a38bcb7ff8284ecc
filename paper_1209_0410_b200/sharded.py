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
"""
from __future__ import annotations

import numpy as np

from .multicurves import MulticurvesIndex, ProjectionScheme, View, gen_rows, merge_packed


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


class ShardedIndex:
    """One rank's share of a G-way sharded Multicurves index."""

    def __init__(self, local: MulticurvesIndex, rank: int, world: int, group=None):
        self.local = local
        self.rank = rank
        self.world = world
        self.group = group
        self._bufs = {}

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
        import torch
        dev = queries.device
        nq = int(queries.shape[0])
        if self.world == 1:
            return self.local.search_batch(queries, k, shard_depth, out=out)
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
