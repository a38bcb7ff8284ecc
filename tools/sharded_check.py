"""torchrun --nproc-per-node G tools/sharded_check.py : NCCL sharded search on G
GPUs (per-shard sm_100a search + all-gather + K4 merge) against the sharded
CPU oracle.  Rank 0 prints 'sharded ok' on bit-identical results."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.sharded import ShardedIndex  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n, nq, k = 20000, 64, 10
scheme = H.default_scheme(128, 8, 16)
sidx = ShardedIndex.from_generator(n, scheme, H.LIFTED, rank, world, local)
qs = H.gen_queries(0, nq, n, device=local)
bad = 0
for depth in (64, H.shard_probe_depth(350, world)):
    ids, sq, ln = sidx.search(qs, k, depth)
    torch.cuda.synchronize()
    if rank == 0:
        from oracle import pyoracle as P
        rows = P.gen_rows(0, n)
        oids, odist, oln = P.sharded_search(H.LIFTED.floats(rows), H.LIFTED.floats(qs.cpu().numpy()), world, 8, 16,
                                            k, depth)
        got_ids, got_sq, got_ln = ids.cpu().numpy(), sq.cpu().numpy(), ln.cpu().numpy()
        bad += int(not np.array_equal(got_ln, oln))
        for q in range(nq):
            L = int(oln[q])
            bad += int(not np.array_equal(got_ids[q, :L], oids[q, :L]))
            d = np.sqrt(got_sq[q, :L].astype(np.float64)) / 256.0
            bad += int(d.tobytes() != odist[q, :L].tobytes())
    # every rank holds the same merged result
    t = ids.view(torch.int64).sum().reshape(1)
    tt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(tt, t)
    bad += int(any(int(x.item()) != int(t.item()) for x in tt))
# exact brute force across shards
ex_ids, _, _ = sidx.brute_force(qs[:16], k)
if rank == 0:
    from oracle import pyoracle as P
    rows = P.gen_rows(0, n)
    bids, _, _ = P.brute_force(H.LIFTED.floats(rows), H.LIFTED.floats(qs[:16].cpu().numpy()), k)
    bad += int(not np.array_equal(ex_ids.cpu().numpy(), bids))
    print("sharded ok" if bad == 0 else f"sharded FAILED ({bad})", flush=True)
dist.destroy_process_group()
sys.exit(1 if bad else 0)
