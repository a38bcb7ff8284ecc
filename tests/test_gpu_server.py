"""The C++ batch-size controller (hcg_server_*, csrc/serve.cpp; DTAHE Alg. 3
without the CPU branch) on a B200:
every query answered exactly once with the search's own results (work
conservation and correctness independence), FIFO batches,
batch size following the load, response times covering H2D + search + D2H,
and the online submit / wait path from several threads."""
import threading

import numpy as np
import pytest

from hcg_testutil import gpu_available
from oracle import pyoracle as P

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200.controller import poisson_arrivals  # noqa: E402
from paper_1209_0410_b200.server import Server  # noqa: E402

N, K, D = 30000, 10, 350


@pytest.fixture(scope="module")
def index():
    return H.MulticurvesIndex(P.gen_rows(0, N), H.default_scheme(128, 8, 16), H.LIFTED)


@pytest.fixture(scope="module")
def queries():
    return P.gen_queries(0, 6000, N)


def _direct(index, q):
    return index.search_batch(q, K, D)


def test_burst_fills_batches_and_matches_search(index, queries):
    srv = Server(index, K, D, max_batch=1024, slots=2)
    ids, sq, ln, lat, sizes = srv.replay(queries, np.zeros(len(queries)))
    ri, rs, rl = _direct(index, queries)
    np.testing.assert_array_equal(ids, ri)
    np.testing.assert_array_equal(sq, rs)
    np.testing.assert_array_equal(ln, rl)
    assert sizes.sum() == len(queries)           # each query exactly once
    assert sizes.max() == 1024 and (sizes[:-1] == 1024).sum() >= len(sizes) - 2  # saturation: full buffers
    assert (lat > 0).all()
    # FIFO: completion times never decrease along the arrival order (batches are contiguous and in order)
    assert np.all(np.diff(lat) >= -1e-9)
    srv.close()


def test_light_load_gives_small_batches(index, queries):
    srv = Server(index, K, D, max_batch=8192, slots=2)
    q = queries[:600]
    arr = poisson_arrivals(20_000.0, len(q), seed=3)  # 50 us apart: far below capacity
    ids, sq, ln, lat, sizes = srv.replay(q, arr)
    ri, rs, rl = _direct(index, q)
    np.testing.assert_array_equal(ids, ri)
    np.testing.assert_array_equal(sq, rs)
    assert sizes.sum() == len(q)
    assert np.median(sizes) <= 4     # the device-idle rule launches (almost) every query on its own
    assert np.median(lat) < 2e-3     # one small search + PCIe both ways
    srv.close()


@pytest.mark.parametrize("slots,rate", [(2, 1e6), (4, 3e6), (8, 6e6)])
def test_side_by_side_batches_match_search(index, queries, slots, rate):
    """Light-to-middle load: small batches run side by side on their slots'
    own streams, larger ones through the pipeline after them (serve.cpp pick);
    every query is answered once with hcg_search's exact results."""
    srv = Server(index, K, D, max_batch=8192, slots=slots)
    q = queries[:6000]
    ids, sq, ln, lat, sizes = srv.replay(q, poisson_arrivals(rate, len(q), seed=slots))
    ri, rs, rl = _direct(index, q)
    np.testing.assert_array_equal(ids, ri)
    np.testing.assert_array_equal(sq, rs)
    np.testing.assert_array_equal(ln, rl)
    assert sizes.sum() == len(q) and (lat > 0).all()
    srv.close()


def test_min_batch_and_max_wait_buffer_queries(index, queries):
    """min_batch=64 with max_wait 2 ms: while a batch is in flight, arrivals
    are held until 64 wait or the oldest waited 2 ms."""
    srv = Server(index, K, D, max_batch=8192, min_batch=64, max_wait=2e-3, slots=2)
    q = queries[:2000]
    arr = poisson_arrivals(400_000.0, len(q), seed=4)
    ids, sq, ln, lat, sizes = srv.replay(q, arr)
    ri, _, _ = _direct(index, q)
    np.testing.assert_array_equal(ids, ri)
    assert sizes.sum() == len(q)
    srv.close()


def test_online_submit_wait_threads(index, queries):
    srv = Server(index, K, D, max_batch=512, slots=2)
    srv.start(capacity=4096)
    ri, rs, rl = _direct(index, queries[:3000])
    errors = []

    def client(lo, hi, step):
        try:
            for s in range(lo, hi, step):
                t = srv.submit(queries[s:s + step])
                ids, sq, ln, lat = srv.wait(t)
                assert np.array_equal(ids, ri[s:s + step]) and np.array_equal(sq, rs[s:s + step])
                assert (lat > 0).all()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=client, args=(i * 1000, (i + 1) * 1000, st)) for i, st in enumerate((1, 37, 250))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    srv.close()


def test_server_validation(index):
    with pytest.raises(H.HcgInvalidArgument):
        Server(index, 0, D)
    with pytest.raises(H.HcgInvalidArgument):
        Server(index, K, D, slots=0)
    srv = Server(index, K, D)
    with pytest.raises(H.HcgInvalidArgument):
        srv.replay(np.zeros((3, 128), np.uint8), np.array([0.0, 2.0, 1.0]))  # arrivals must not decrease
    srv.close()


def test_server_over_a_shard_group(queries):
    """One process, all GPUs: the server dispatches to a shard group (per-GPU
    search, NCCL all-gather, merge); results equal the group's direct search
    and the sharded oracle."""
    import torch
    G = min(torch.cuda.device_count(), 4)
    if G < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_1209_0410_b200.sharded import ShardGroup
    rows = P.gen_rows(0, N)
    grp = ShardGroup.build(rows, H.default_scheme(128, 8, 16), H.LIFTED, list(range(G)))
    depth = H.shard_probe_depth(D, G)
    srv = Server(grp, K, depth, max_batch=2048)
    q = queries[:3000]
    ids, sq, ln, lat, sizes = srv.replay(q, poisson_arrivals(2e6, len(q), seed=5))
    gi, gs, gl = grp.search(q, K, depth)
    np.testing.assert_array_equal(ids, gi)
    np.testing.assert_array_equal(sq, gs)
    oids, odist, oln = P.sharded_search(H.LIFTED.floats(rows), H.LIFTED.floats(q[:200]), G, 8, 16, K, depth)
    np.testing.assert_array_equal(ids[:200], oids)
    assert sizes.sum() == len(q)
    srv.close()
    grp.close()
