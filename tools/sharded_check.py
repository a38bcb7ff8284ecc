"""torchrun --nproc-per-node G tools/sharded_check.py [--n N] [--queries Q] :
sharded search on G GPUs through libhcg's shard group (hcg_shard_group_*:
per-shard sm_100a search + NCCL all-gather inside the library + K4 merge)
against the reference's sharded search.

The reference side: for n <= 200K the independent oracle's sharded search
(floats), and for every n the reference's own TUs (oracle/_ref, one
hc::MulticurvesIndex per shard with the shard's global ids, searched at the
per-shard depth, merged by (distance, id)) when they are available.  The
torch.distributed aggregate (search_torch) must agree too, and every rank
must hold the same merged result.  Rank 0 prints one JSON line and
'sharded ok' on bit-identical results."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.sharded import ShardedIndex  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=20000)
p.add_argument("--queries", type=int, default=64)
p.add_argument("--view", choices=["lifted", "raw"], default="lifted")
p.add_argument("--depths", default="")
p.add_argument("--k", type=int, default=10)
a = p.parse_args()

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n, nq, k = a.rows, a.queries, a.k
view, m = (H.LIFTED, 16) if a.view == "lifted" else (H.RAW, 8)
scheme = H.default_scheme(128, 8, m)
t0 = time.time()
sidx = ShardedIndex.from_generator(n, scheme, view, rank, world, local)
torch.cuda.synchronize()
build_s = time.time() - t0
qs = H.gen_queries(0, nq, n, device=local)
depths = [int(x) for x in a.depths.split(",") if x] or [64, H.shard_probe_depth(350, world)]
bad = 0
report = {"n": n, "shards": world, "queries": nq, "k": k, "view": a.view, "depths": depths, "build_s": round(build_s, 2),
          "checks": []}
ref_tus = {}
if rank == 0:
    from oracle import pyoracle as P
    if P.ref_available():
        t1 = time.time()
        ref_tus = P.ref_sharded_search(n, world, qs.cpu().numpy(), 8, m, 1, 1 if a.view == "lifted" else 0, k, depths)
        report["reference_tus_s"] = round(time.time() - t1, 1)
dist.barrier()
for depth in depths:
    ids, sq, ln = sidx.search(qs, k, depth)              # libhcg shard group
    tids, tsq, tln = sidx.search_torch(qs, k, depth)     # torch.distributed aggregate
    torch.cuda.synchronize()
    same_torch = torch.equal(ids, tids) and torch.equal(sq, tsq) and torch.equal(ln, tln)
    bad += int(not same_torch)
    # the routed aggregate: this rank's block of the batch equals the full result's rows
    (rids, rsq, rln), first, cnt = sidx.shard_group.search_routed(qs, k, depth)
    torch.cuda.synchronize()
    blk = slice(first, first + cnt)
    same_routed = (torch.equal(rids[blk], ids[blk]) and torch.equal(rsq[blk], sq[blk]) and torch.equal(rln[blk], ln[blk])
                   and cnt == (nq * (rank + 1)) // world - (nq * rank) // world)
    bad += int(not same_routed)
    # every rank holds the same merged result
    t = ids.view(torch.int64).sum().reshape(1)
    tt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(tt, t)
    bad += int(any(int(x.item()) != int(t.item()) for x in tt))
    if rank == 0:
        from oracle import pyoracle as P
        got_ids, got_sq, got_ln = ids.cpu().numpy(), sq.cpu().numpy(), ln.cpu().numpy()
        refs = []
        if n <= 200_000:
            rows = P.gen_rows(0, n)
            refs.append(("oracle", P.sharded_search(view.floats(rows), view.floats(qs.cpu().numpy()), world, 8, m, k,
                                                    depth)))
        if depth in ref_tus:
            refs.append(("reference_tus", ref_tus[depth]))
        for name, (oids, odist, oln) in refs:
            mism = int((got_ln != oln).sum())
            for q in range(nq):
                L = int(oln[q])
                d = np.sqrt(got_sq[q, :L].astype(np.float64)) * view.scale
                if not (np.array_equal(got_ids[q, :L], oids[q, :L]) and d.tobytes() == odist[q, :L].tobytes()):
                    mism += 1
            bad += mism
            report["checks"].append({"depth": depth, "against": name, "mismatched_queries": mism,
                                     "torch_aggregate_identical": bool(same_torch),
                                     "routed_block_identical_rank0": bool(same_routed)})
dist.barrier()
# exact brute force across shards
ex_ids, _, _ = sidx.brute_force(qs[:16], k)
if rank == 0 and n <= 200_000:
    from oracle import pyoracle as P
    rows = P.gen_rows(0, n)
    bids, _, _ = P.brute_force(view.floats(rows), view.floats(qs[:16].cpu().numpy()), k)
    bad += int(not np.array_equal(ex_ids.cpu().numpy(), bids))
if rank == 0:
    report["ok"] = bad == 0
    print(json.dumps(report), flush=True)
    print("sharded ok" if bad == 0 else f"sharded FAILED ({bad})", flush=True)
dist.barrier()
sidx.shard_group.close()
dist.destroy_process_group()
sys.exit(1 if bad else 0)
