"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bit-exact on every observable the reference exposes: curve keys, sorted
subindexes (key, id order), rank_of / window, deduplicated candidate sets,
top-k ids and distances (the rooted double the reference returns).
"""
import numpy as np
import pytest

from oracle import pyoracle as P
from hcg_testutil import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402

VIEWS = [(H.RAW, 8), (H.LIFTED, 16)]


def _oracle(rows, view, curves, m, kind, scheme=None, ids=None):
    f = view.floats(rows)
    if scheme is None:
        return P.Oracle(f, curves, m, kind, ids=ids)
    off = np.cumsum([0] + [len(a) for a in scheme.assignment]).astype(np.uint32)
    asg = np.concatenate([np.asarray(a, np.uint32) for a in scheme.assignment])
    return P.Oracle(f, curves, m, kind, ids=ids, off=off, assign=asg)


def _check_search(gi, oi, view, qs, k, depth):
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(view.floats(qs), k, depth)
    np.testing.assert_array_equal(ln, oln)
    d = gi.rooted(sq)
    for q in range(qs.shape[0]):
        L = int(ln[q])
        np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
        # bit-exact doubles (integer squared distances are exact)
        assert d[q, :L].tobytes() == odist[q, :L].tobytes(), (q, d[q, :L], odist[q, :L])
        assert (ids[q, L:] == np.uint64(2**64 - 1)).all()


@pytest.mark.parametrize("view,m", VIEWS, ids=["raw", "lifted"])
@pytest.mark.parametrize("kind", [H.HILBERT, H.ZORDER], ids=["hilbert", "zorder"])
@pytest.mark.parametrize("curves", [1, 2, 4, 8, 16])
def test_keys_sorted_windows_search(view, m, kind, curves):
    if (128 // curves) * m > 1024:
        pytest.skip("key wider than HC_MAX_KEY_BITS (the reference rejects it too)")
    n, nq = 3000, 48
    rows = P.gen_rows(0, n)
    qs = P.gen_queries(0, nq, n)
    scheme = H.default_scheme(128, curves, m, kind)
    gi = H.MulticurvesIndex(rows, scheme, view)
    oi = _oracle(rows, view, curves, m, kind)
    f = view.floats(rows)
    for c in range(curves):
        # keys of arbitrary rows (curve_encode(project(v, c)))
        gk = gi.keys(rows[:200], c)
        w = gk.shape[1]
        ok = np.stack([oi.query_key(f[i], c)[:w] for i in range(200)])
        np.testing.assert_array_equal(gk, ok)
        # sorted subindex: (key, id) order, keys re-expanded from the suffix store
        gids, gkeys = gi.subindex(c, with_keys=True)
        okeys, oids = oi.sorted(c)
        np.testing.assert_array_equal(gids, oids)
        np.testing.assert_array_equal(gkeys, okeys)
    for depth in (1, 7, 64, 350):
        r, b, e = gi.windows(qs, depth)
        orr, ob, oe = oi.windows(view.floats(qs), depth)
        np.testing.assert_array_equal(r, orr)
        np.testing.assert_array_equal(b, ob)
        np.testing.assert_array_equal(e, oe)
        cands = gi.candidates(qs[:16], depth)
        for q in range(16):
            np.testing.assert_array_equal(cands[q], oi.candidates(view.floats(qs[q]), depth))
        _check_search(gi, oi, view, qs, 10, depth)


@pytest.mark.parametrize("view,m", VIEWS, ids=["raw", "lifted"])
@pytest.mark.parametrize("k", [1, 10, 33, 100, 256])
def test_search_k_sweep(view, m, k):
    n, nq = 4000, 40
    rows = P.gen_rows(100, n)
    qs = P.gen_queries(7, nq, n)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, m), view)
    oi = _oracle(rows, view, 8, m, H.HILBERT)
    for depth in (16, 350):
        _check_search(gi, oi, view, qs, k, depth)


def test_uniform_bytes_ties_and_uneven_scheme():
    rng = np.random.default_rng(5)
    for d_full, curves, m in ((20, 3, 8), (100, 7, 16), (130, 5, 8), (128, 1, 8)):
        rows = rng.integers(0, 256, (1500, d_full), dtype=np.uint8)
        rows[700:760] = rows[10]  # exact duplicates: ties broken by id everywhere
        qs = rng.integers(0, 256, (30, d_full), dtype=np.uint8)
        qs[:5] = rows[[10, 0, 1499, 700, 3]]
        scheme = H.default_scheme(d_full, curves, m)
        for view in (H.RAW, H.LIFTED):
            gi = H.MulticurvesIndex(rows, scheme, view)
            oi = _oracle(rows, view, curves, m, H.HILBERT, scheme=scheme)
            for c in range(curves):
                gids, gkeys = gi.subindex(c, with_keys=True)
                okeys, oids = oi.sorted(c)
                np.testing.assert_array_equal(gids, oids)
                np.testing.assert_array_equal(gkeys, okeys)
            for depth in (3, 50, 2000):
                _check_search(gi, oi, view, qs, 12, depth)


def test_very_large_candidate_sets():
    """curves x depth beyond the shared-memory union (global CAS table path)."""
    rows = P.gen_rows(0, 6000)
    qs = P.gen_queries(0, 24, 6000)
    for curves, m, depth in ((16, 8, 5000), (8, 16, 4096)):
        gi = H.MulticurvesIndex(rows, H.default_scheme(128, curves, m), H.LIFTED if m == 16 else H.RAW)
        view = H.LIFTED if m == 16 else H.RAW
        oi = _oracle(rows, view, curves, m, H.HILBERT)
        _check_search(gi, oi, view, qs, 10, depth)
        _check_search(gi, oi, view, qs, 100, depth)
        cands = gi.candidates(qs[:3], depth)
        for q in range(3):
            np.testing.assert_array_equal(cands[q], oi.candidates(view.floats(qs[q]), depth))


def test_tiny_and_empty_indexes():
    rows = P.gen_rows(0, 5)
    qs = P.gen_queries(0, 4, 5)
    for n in (0, 1, 2, 5):
        gi = H.MulticurvesIndex(rows[:n], H.default_scheme(128, 8, 8), H.RAW)
        assert gi.size() == n
        ids, sq, ln = gi.search_batch(qs, 10, 350)
        assert (ln == n).all()
        if n:
            oi = _oracle(rows[:n], H.RAW, 8, 8, H.HILBERT)
            _check_search(gi, oi, H.RAW, qs, 10, 350)
        else:
            assert (ids == np.uint64(2**64 - 1)).all()


def test_self_query_distance_zero():
    """q equal to an indexed vector, any depth >= 1, k=1."""
    rows = P.gen_rows(0, 2000)
    for view, m in VIEWS:
        gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, m), view)
        for i in (0, 17, 1999):
            nl = gi.search(rows[i], H.SearchParams(k=1, probe_depth=1))
            assert nl[0].distance == 0.0
            assert np.array_equal(rows[nl[0].id], rows[i])


def test_one_curve_full_depth_is_brute_force():
    """curves=1 and depth >= n is identical to brute_force_knn."""
    rows = P.gen_rows(3, 1500)
    qs = P.gen_queries(0, 20, 1500)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 1, 8), H.RAW)
    ids, sq, ln = gi.search_batch(qs, 10, 1500)
    bids, bdist, bln = P.brute_force(H.RAW.floats(rows), H.RAW.floats(qs), 10)
    np.testing.assert_array_equal(ids, bids)
    assert gi.rooted(sq).tobytes() == bdist.tobytes()


def test_brute_force_kernel():
    rows = P.gen_rows(0, 70000)  # > one 32768-row chunk
    qs = P.gen_queries(0, 37, 70000)
    for view, m in VIEWS:
        gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, m), view)
        for k in (1, 10, 100):
            ids, sq, ln = gi.brute_force(qs, k)
            bids, bdist, bln = P.brute_force(view.floats(rows), view.floats(qs), k)
            np.testing.assert_array_equal(ln, bln)
            np.testing.assert_array_equal(ids, bids)
            assert gi.rooted(sq).tobytes() == bdist.tobytes()


def test_generator_matches_oracle():
    import torch
    g = H.gen_rows(0, 3000).cpu().numpy()
    np.testing.assert_array_equal(g, P.gen_rows(0, 3000))
    g = H.gen_rows(5, 1000, stride=7).cpu().numpy()
    o = P.gen_rows(0, 7 * 1000 + 5)[5::7][:1000]
    np.testing.assert_array_equal(g, o)
    q = H.gen_queries(11, 500, 123456).cpu().numpy()
    np.testing.assert_array_equal(q, P.gen_queries(11, 500, 123456))
    del torch


def test_device_and_host_buffers_agree():
    import torch
    rows = P.gen_rows(0, 5000)
    qs = P.gen_queries(0, 64, 5000)
    gi = H.MulticurvesIndex(torch.from_numpy(rows).cuda(), H.default_scheme(128, 8, 16), H.LIFTED)
    ids_h, sq_h, ln_h = gi.search_batch(qs, 10, 350)
    ids_d, sq_d, ln_d = gi.search_batch(torch.from_numpy(qs).cuda(), 10, 350)
    assert ids_d.is_cuda
    np.testing.assert_array_equal(ids_h, ids_d.cpu().numpy())
    np.testing.assert_array_equal(sq_h, sq_d.cpu().numpy())
    # pinned host buffers
    qp = torch.from_numpy(qs).pin_memory()
    ids_p, sq_p, ln_p = gi.search_batch(qp, 10, 350)
    np.testing.assert_array_equal(ids_h, ids_p)


@pytest.mark.parametrize("shards", [2, 3, 4])
def test_sharded_merge_matches_sharded_oracle(shards):
    """hypershard partition (id mod G) + per-shard search + (dist, id) merge
     against the sharded CPU oracle."""
    import torch
    n, nq, k, depth = 6000, 50, 10, 120
    rows = P.gen_rows(0, n)
    qs = P.gen_queries(0, nq, n)
    view, m = H.LIFTED, 16
    parts = []
    for r in range(shards):
        gi = H.MulticurvesIndex(rows[r::shards], H.default_scheme(128, 8, m), view,
                                id_base=r, id_stride=shards)
        parts.append(gi.search_packed(torch.from_numpy(qs).cuda(), k, depth))
    ids, sq, ln = H.merge_packed(torch.stack(parts), k)
    oids, odist, oln = P.sharded_search(view.floats(rows), view.floats(qs), shards, 8, m, k, depth)
    np.testing.assert_array_equal(ln.cpu().numpy(), oln)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids)
    d = np.sqrt(sq.cpu().numpy().astype(np.float64)) * view.scale
    assert d.tobytes() == odist.tobytes()


def test_error_behaviour():
    rows = P.gen_rows(0, 100)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 8), H.RAW)
    with pytest.raises(ValueError):
        gi.search_batch(rows[:2], 0, 10)       # k must be >= 1
    with pytest.raises(ValueError):
        gi.search_batch(rows[:2], 10, 0)       # probe_depth must be >= 1
    with pytest.raises(ValueError):
        gi.search_batch(rows[:2, :64], 10, 10)  # dimension mismatch
    with pytest.raises(ValueError):
        H.MulticurvesIndex(rows, H.default_scheme(128, 1, 16), H.RAW)  # 2048-bit key > capacity


def test_host_pipeline_matches_direct_search():
    """pipeline.HostPipeline (overlapped H2D / search / D2H) returns exactly the
    per-batch results of search_batch."""
    import torch
    from paper_1209_0410_b200.pipeline import HostPipeline
    rows = P.gen_rows(0, 20000)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    batches = [torch.from_numpy(P.gen_queries(b * 500, 500 - 37 * (b % 3), 20000)).pin_memory() for b in range(6)]
    outs = [(torch.empty((len(q), 10), dtype=torch.uint64).pin_memory(),
             torch.empty((len(q), 10), dtype=torch.uint32).pin_memory(),
             torch.empty((len(q),), dtype=torch.uint32).pin_memory()) for q in batches]
    HostPipeline(lambda q, out: gi.search_batch(q, 10, 350, out=out), 10, 500).run(batches, outs)
    for q, (ids, sq, ln) in zip(batches, outs):
        wi, ws, wl = gi.search_batch(q.numpy(), 10, 350)
        np.testing.assert_array_equal(ids.numpy(), wi)
        np.testing.assert_array_equal(sq.numpy(), ws)
        np.testing.assert_array_equal(ln.numpy(), wl)


@pytest.mark.parametrize("view,m", VIEWS, ids=["raw", "lifted"])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_large_batch_paths(view, m, k):
    """Batches large enough for the warp-per-query gather, the curve-0 batch
    order and (k <= 32, 128-B rows) the row-sketch filter: bit-exact vs the
    oracle, ties included (duplicated rows)."""
    n, nq = 30_000, 20_000
    rows = P.gen_rows(0, n)
    rows[1000:1100] = rows[5]  # exact ties
    qs = P.gen_queries(0, nq, n)
    qs[:50] = rows[5]
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, m), view)
    oi = _oracle(rows, view, 8, m, H.HILBERT)
    _check_search(gi, oi, view, qs, k, 350)
    if k == 10:  # the sorted two-phase locate of large batches
        r, b, e = gi.windows(qs, 350)
        orr, ob, oe = oi.windows(view.floats(qs), 350)
        np.testing.assert_array_equal(r, orr)
        np.testing.assert_array_equal(b, ob)


def test_concurrent_searches_from_threads():
    """search is const and may run concurrently -- four host
    threads, each on its own CUDA stream, get the single-threaded results."""
    import threading
    import torch
    rows = P.gen_rows(0, 20_000)
    qs = P.gen_queries(0, 80_000, 20_000)  # 20K per thread: warp-per-query gather + batch order
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    want = [gi.search_batch(qs[i::4], 10, 200) for i in range(4)]
    got = [None] * 4
    errors = []

    def work(i):
        try:
            st = torch.cuda.Stream()
            q = torch.from_numpy(np.ascontiguousarray(qs[i::4])).cuda()
            for _ in range(3):
                with torch.cuda.stream(st):
                    out = gi.search_batch(q, 10, 200, stream=st)
            st.synchronize()
            got[i] = tuple(t.cpu().numpy() for t in out)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(4):
        for a, b in zip(got[i], want[i]):
            np.testing.assert_array_equal(a, b)


def test_chunked_batches_match_small_batches():
    """A batch whose candidate lists exceed the 2 GB list budget is searched
    in chunks (no batch order); results equal searching slices of it."""
    import torch
    n, nq, depth = 200_000, 60_000, 2000  # 8 curves x 2000 -> 16K ids per query: 3 chunks
    rows = H.gen_rows(0, n)
    qs = H.gen_queries(0, nq, n)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    ids, sq, ln = gi.search_batch(qs, 10, depth)
    for s in (0, 25_000, 59_000):
        i2, s2, l2 = gi.search_batch(qs[s:s + 1000].contiguous(), 10, depth)
        assert torch.equal(ids[s:s + 1000], i2) and torch.equal(sq[s:s + 1000], s2) and torch.equal(ln[s:s + 1000], l2)
