"""Randomised parity: schemes, sizes, depths, k and views drawn at random
(seeded), each search bit-exact against the oracle.  Reaches the rarely used
paths (uneven assignments, wide keys, JMAX 16-32 unions, shared-memory and
global-table unions, 128-thread unions, CTA and warp gathers, the union-less
gather for large batches, k up to 256)."""
import numpy as np
import pytest

from oracle import pyoracle as P
from hcg_testutil import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402


def _random_scheme(rng, d_full, curves):
    perm = rng.permutation(d_full)
    cuts = np.sort(rng.choice(np.arange(1, d_full), curves - 1, replace=False)) if curves > 1 else []
    parts = np.split(perm, cuts)
    return [sorted(int(x) for x in p) for p in parts]


@pytest.mark.parametrize("seed", range(40))
def test_random_configurations(seed):
    rng = np.random.default_rng(1000 + seed)
    d_full = int(rng.choice([16, 24, 64, 100, 128]))
    m = int(rng.choice([4, 8, 12, 16]))
    curves = int(rng.integers(1, min(d_full, 16) + 1))
    assignment = _random_scheme(rng, d_full, curves)
    if max(len(a) for a in assignment) * m > 1024 or max(len(a) for a in assignment) > 128:
        pytest.skip("key wider than HC_MAX_KEY_BITS")
    kind = int(rng.integers(0, 2))
    view = H.LIFTED if rng.random() < 0.5 else H.RAW
    n = int(rng.integers(1, 30_000))
    nq = int(rng.choice([1, 7, 300, 3000, 5000]))
    depth = int(rng.choice([1, 3, 50, 350, 1000, 3000]))
    k = int(rng.choice([1, 10, 33, 100, 256]))
    rows = rng.integers(0, 256, (n, d_full), dtype=np.uint8)
    if n > 50:
        rows[n // 2:n // 2 + 20] = rows[0]  # ties
    qs = rng.integers(0, 256, (nq, d_full), dtype=np.uint8)
    scheme = H.ProjectionScheme(d_full, m, kind, 0, assignment)
    gi = H.MulticurvesIndex(rows, scheme, view)
    off = np.cumsum([0] + [len(a) for a in assignment]).astype(np.uint32)
    asg = np.concatenate([np.asarray(a, np.uint32) for a in assignment])
    oi = P.Oracle(view.floats(rows), curves, m, kind, off=off, assign=asg)
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(view.floats(qs), k, depth)
    np.testing.assert_array_equal(ln, oln)
    d = gi.rooted(sq)
    for q in range(nq):
        L = int(ln[q])
        np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
        assert d[q, :L].tobytes() == odist[q, :L].tobytes()
    for q in range(min(nq, 3)):
        np.testing.assert_array_equal(gi.candidates(qs[q], depth)[0], oi.candidates(view.floats(qs[q]), depth))


@pytest.mark.parametrize("seed", range(12))
def test_random_configurations_f32(seed):
    """The same over float rows: keys, candidates, ids and distances bit-exact
    (sequential double sums in index order, as vecio.cpp:87-95)."""
    rng = np.random.default_rng(5000 + seed)
    d_full = int(rng.choice([16, 24, 64, 100, 128]))
    m = int(rng.choice([8, 16, 32]))
    curves = int(rng.integers(1, min(d_full, 16) + 1))
    assignment = _random_scheme(rng, d_full, curves)
    if max(len(a) for a in assignment) * m > 1024:
        pytest.skip("key wider than HC_MAX_KEY_BITS")
    kind = int(rng.integers(0, 2))
    n = int(rng.integers(1, 20_000))
    nq = int(rng.choice([1, 64, 3000, 17_000]))
    depth = int(rng.choice([1, 50, 350, 2000]))
    k = int(rng.choice([1, 10, 64]))
    rows = (rng.standard_normal((n, d_full)) * rng.choice([1e-3, 1.0, 1e3])).astype(np.float32)
    qs = (rng.standard_normal((nq, d_full)) * 1.0).astype(np.float32)
    scheme = H.ProjectionScheme(d_full, m, kind, 0, assignment)
    gi = H.MulticurvesIndex(rows, scheme)
    off = np.cumsum([0] + [len(a) for a in assignment]).astype(np.uint32)
    asg = np.concatenate([np.asarray(a, np.uint32) for a in assignment])
    oi = P.Oracle(rows, curves, m, kind, off=off, assign=asg)
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(qs, k, depth)
    np.testing.assert_array_equal(ln, oln)
    d = gi.rooted(sq)
    for q in range(nq):
        L = int(ln[q])
        np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
        assert d[q, :L].tobytes() == odist[q, :L].tobytes()


@pytest.mark.parametrize("seed", range(16))
def test_random_configurations_large_batch(seed):
    """>= 16K queries with k <= 128: the union-less gather (k_gather_nu walks the
    C windows, queues its offers and merges + dedups a full queue; list
    widths R = 1 / 2 / 4 / 8 switch at k = 16 / 48 / 112) over random schemes,
    row widths, depths (windows past both ends included) and views."""
    rng = np.random.default_rng(9000 + seed)
    d_full = int(rng.choice([16, 24, 64, 100, 128]))
    m = int(rng.choice([8, 16]))
    curves = int(rng.integers(1, min(d_full, 16) + 1))
    assignment = _random_scheme(rng, d_full, curves)
    if max(len(a) for a in assignment) * m > 1024:
        pytest.skip("key wider than HC_MAX_KEY_BITS")
    kind = int(rng.integers(0, 2))
    view = H.LIFTED if rng.random() < 0.5 else H.RAW
    n = int(rng.integers(1, 12_000))
    nq = int(rng.choice([16_384, 17_001]))
    depth = int(rng.choice([1, 3, 50, 350, 2000]))
    k = int(rng.choice([1, 10, 16, 17, 32, 33, 48, 49, 64, 96, 100, 112, 113, 128]))
    rows = rng.integers(0, 256, (n, d_full), dtype=np.uint8)
    if n > 50:
        rows[n // 2:n // 2 + 20] = rows[0]  # ties and repeats across curves
    qs = rng.integers(0, 256, (nq, d_full), dtype=np.uint8)
    qs[:64] = rows[rng.integers(0, n, 64)]  # self queries
    scheme = H.ProjectionScheme(d_full, m, kind, 0, assignment)
    gi = H.MulticurvesIndex(rows, scheme, view)
    off = np.cumsum([0] + [len(a) for a in assignment]).astype(np.uint32)
    asg = np.concatenate([np.asarray(a, np.uint32) for a in assignment])
    oi = P.Oracle(view.floats(rows), curves, m, kind, off=off, assign=asg)
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(view.floats(qs), k, depth)
    np.testing.assert_array_equal(ln, oln)
    d = gi.rooted(sq)
    for q in range(nq):
        L = int(ln[q])
        np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
        assert d[q, :L].tobytes() == odist[q, :L].tobytes()
        assert (ids[q, L:] == np.uint64(2**64 - 1)).all()


@pytest.mark.parametrize("k,depth", [(16, 1100), (17, 300), (32, 260), (33, 1100), (48, 300), (49, 300), (64, 260), (65, 520), (100, 600),
                                     (112, 1100), (113, 800), (128, 1100)])
def test_unionless_wide_k_long_walks(k, depth):
    """k > 16 on walks of C x depth >= 2048 (4096 for k > 64, 6144 for k > 112) and >= 16K
    queries: the union-less walk with queued offers, merged and deduplicated
    per full queue, at every list width and both sides of each switch."""
    n = 12_000
    rows = P.gen_rows(0, n)
    qs = P.gen_queries(0, 16_384, n)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    assert gi.unionless(16_384, k, depth)
    oi = P.Oracle(H.LIFTED.floats(rows), 8, 16)
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(H.LIFTED.floats(qs), k, depth)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(ids, oids)
    assert gi.rooted(sq).tobytes() == odist.tobytes()


@pytest.mark.parametrize("k", [10, 40, 100])
def test_unionless_many_ties(k):
    """Rows of 0 / 1 bytes: most distances tie, so many offers sit exactly at
    the k-th distance -- they pass the queue's distance-only filter and the
    merge orders them by id (vecio.cpp:102-105)."""
    rng = np.random.default_rng(77 + k)
    n = 6000
    rows = rng.integers(0, 2, (n, 128), dtype=np.uint8)
    rows[100:400] = rows[0]  # exact repeats as well
    qs = rng.integers(0, 2, (16_384, 128), dtype=np.uint8)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    assert gi.unionless(16_384, k, 700)
    oi = P.Oracle(H.LIFTED.floats(rows), 8, 16)
    ids, sq, ln = gi.search_batch(qs, k, 700)
    oids, odist, oln = oi.search(H.LIFTED.floats(qs), k, 700)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(ids, oids)
    assert gi.rooted(sq).tobytes() == odist.tobytes()


@pytest.mark.parametrize("view,m", [(H.LIFTED, 16), (H.RAW, 8)])
def test_batch_size_paths_agree(view, m):
    """The fused one-CTA-per-query latency kernel (<= 512 queries), the
    union + gather path and the union-less walk (>= 16K) return the same
    lists for the same queries."""
    n = 30_000
    rows = P.gen_rows(0, n)
    qs = P.gen_queries(0, 16_384, n)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, m), view)
    for k, depth in ((10, 350), (100, 350), (1, 16), (256, 600)):
        big = gi.search_batch(qs, k, depth)
        for lo, hi in ((0, 1), (5, 37), (100, 612), (1000, 4000)):
            part = gi.search_batch(qs[lo:hi], k, depth)
            for x, y in zip(part, big):
                np.testing.assert_array_equal(x, y[lo:hi] if y.ndim == 1 else y[lo:hi])
