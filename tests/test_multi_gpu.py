"""Sharded search on >= 2 GPUs (skipped on a 1-GPU box; the host-side
protocol is covered on CPU by test_sharded_gloo):

* one process per GPU (torchrun): libhcg's shard group joined per rank
  (hcg_shard_group_join) against the sharded CPU oracle and the reference's
  own TUs, and against the torch.distributed aggregate;
* one process over all GPUs: hcb::ShardedIndex (C++, hcg_shard_group_build,
  ncclCommInitAll) against the sharded oracle."""
import os
import subprocess
import sys

import pytest

from hcg_testutil import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


needs2 = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")]


@pytest.mark.parametrize("view,queries", [("lifted", 64), ("raw", 64), ("lifted", 3)])
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")
def test_sharded_search_per_rank_processes(view, queries):
    """Per-rank shard groups vs the sharded oracle and the reference TUs; the
    routed aggregate's blocks (3 queries: some ranks aggregate none) vs the
    all-gathered result."""
    g = min(_ngpus(), 4)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
                          "--master-addr", "127.0.0.1", "--master-port", "29533",
                          os.path.join(ROOT, "tools", "sharded_check.py"), "--view", view, "--queries", str(queries)],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "sharded ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")
def test_cpp_shard_group_single_process():
    binp = os.path.join(ROOT, "tests", "cpp", "test_shard_group.bin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_shard_group.cpp"),
                    "-L", os.path.join(ROOT, "paper_1209_0410_b200"), "-lhcg", "-L", os.path.join(ROOT, "oracle"),
                    "-loracle", "-L", "/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1209_0410_b200')}:{os.path.join(ROOT, 'oracle')}",
                    "-o", binp], check=True)
    out = subprocess.run([binp], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "shard group ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")
def test_one_process_group_with_empty_shards():
    """Fewer rows than GPUs: the empty shards' padding still reaches GPU 0 (the
    fused exchange writes it locally and copies it over), and the merge equals
    the sharded oracle."""
    import numpy as np
    import paper_1209_0410_b200 as H
    from oracle import pyoracle as P
    from paper_1209_0410_b200.sharded import ShardGroup
    G = min(_ngpus(), 4)
    for n in (1, G - 1, G + 1):
        rows = P.gen_rows(0, n)
        qs = P.gen_queries(0, 7, max(n, 1))
        grp = ShardGroup.build(rows, H.default_scheme(128, 8, 16), H.LIFTED, list(range(G)))
        for nq in (7, 3):  # the small-batch kernel and a resized exchange buffer
            ids, sq, ln = grp.search(qs[:nq], 5, 64)
            oids, odist, oln = P.sharded_search(H.LIFTED.floats(rows), H.LIFTED.floats(qs[:nq]), G, 8, 16, 5, 64)
            np.testing.assert_array_equal(ln, oln)
            for q in range(nq):
                L = int(oln[q])
                np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
                assert (np.sqrt(sq[q, :L].astype(np.float64)) / 256.0).tobytes() == odist[q, :L].tobytes()
        grp.close()
