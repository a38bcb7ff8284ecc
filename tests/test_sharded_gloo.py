"""Multi-process sharding on CPU (gloo, world size 2, 3 and 8 -- the 8-GPU box layout): each rank owns the
ids i = rank (mod G), answers every query on its shard, packs
(sqdist << 32 | gid), and the product's exchange() all-gathers the blocks; the
(distance, id) merge of the gathered blocks must equal the sharded oracle
(SURVEY F7).  The per-shard search here is the CPU oracle --
the GPU per-shard search and the K4 merge kernel are covered by -m gpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as P
from paper_1209_0410_b200.sharded import exchange, shard_rows

N, NQ, K, DEPTH = 3000, 12, 10, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = P.gen_rows(rank, shard_rows(N, rank, world), stride=world)
        gid = np.arange(rank, N, world, dtype=np.uint64)
        assert len(gid) == rows.shape[0]
        qs = P.view_floats(P.gen_queries(0, NQ, N), P.LIFTED)
        ids, dist_, ln = P.Oracle(P.view_floats(rows, P.LIFTED), 8, 16, ids=gid).search(qs, K, DEPTH)
        sq = np.rint((dist_ * 256.0) ** 2).astype(np.int64)  # exact: lifted distance^2 = S / 2^16
        packed = (sq << 32) | ids.astype(np.int64)
        packed[np.arange(K)[None, :] >= ln[:, None]] = -1
        gathered = exchange(torch.from_numpy(packed), world)
        if rank == 0:
            q.put(gathered.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_exchange_and_merge_match_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), q), nprocs=world, join=True, start_method="spawn")
    gathered = q.get()
    assert gathered.shape == (world, NQ, K)
    flat = gathered.reshape(world, NQ, K).transpose(1, 0, 2).reshape(NQ, world * K)
    merged = np.sort(flat.view(np.uint64), axis=1)[:, :K]  # (sqdist, id) integer order
    oids, odist, oln = P.sharded_search(P.view_floats(P.gen_rows(0, N), P.LIFTED),
                                        P.view_floats(P.gen_queries(0, NQ, N), P.LIFTED), world, 8, 16, K, DEPTH)
    for qi in range(NQ):
        L = int(oln[qi])
        np.testing.assert_array_equal(merged[qi, :L] & np.uint64(0xFFFFFFFF), oids[qi, :L])
        d = np.sqrt((merged[qi, :L] >> np.uint64(32)).astype(np.float64)) / 256.0
        assert d.tobytes() == odist[qi, :L].tobytes()


def test_partition_is_a_disjoint_cover():
    for n in (0, 1, 7, 1000, 1001):
        for g in (1, 2, 3, 8):
            sizes = [shard_rows(n, r, g) for r in range(g)]
            assert sum(sizes) == n
            assert max(sizes) - min(sizes) <= 1
