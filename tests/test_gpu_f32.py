"""GPU parity for float descriptors (HCG_F32): the reference's own component
type, quantized on the device by float_to_ordinal >> (32 - m)
(curve.cpp:166-174) and scored in double (vecio.cpp:87-95).

Keys, sorted subindexes, windows, candidate sets, top-k ids and rooted
distances are all bit-exact against the oracle: the GPU sums the reference's
double terms (double(a) - double(b))^2 sequentially in index order with
separately rounded subtract / multiply / add, the same double as
squared_distance (vecio.cpp:87-95), so near-ties order as the reference orders them.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as P
from hcg_testutil import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402
from paper_1209_0410_b200._lib import HcgError  # noqa: E402



def float_rows(n, d, seed, scale=40.0):
    """Signed floats over several binades, with exact zeros, -0.0 and duplicates."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((n, d)) * scale).astype(np.float32)
    x[rng.random((n, d)) < 0.05] = 0.0
    x[rng.random((n, d)) < 0.02] = -0.0
    x[:, : d // 4] *= np.float32(1e-3)  # a small-magnitude band
    if n > 20:
        x[10:20] = x[0]  # duplicate rows: equal distances, tie by id
    return x


def _oracle(rows, curves, m, kind):
    return P.Oracle(rows, curves, m, kind)


def _check_search(gi, oi, qs, k, depth, exact=True):
    ids, sq, ln = gi.search_batch(qs, k, depth)
    oids, odist, oln = oi.search(qs, k, depth)
    np.testing.assert_array_equal(ln, oln)
    d = gi.rooted(sq)
    for q in range(qs.shape[0]):
        L = int(ln[q])
        np.testing.assert_array_equal(ids[q, :L], oids[q, :L])
        assert d[q, :L].tobytes() == odist[q, :L].tobytes(), (q, d[q, :L], odist[q, :L])
        assert (ids[q, L:] == np.uint64(2**64 - 1)).all()
        assert np.isinf(sq[q, L:]).all()


@pytest.mark.parametrize("m", [8, 16, 32])
@pytest.mark.parametrize("kind", [H.HILBERT, H.ZORDER], ids=["hilbert", "zorder"])
@pytest.mark.parametrize("curves", [2, 4, 8])
def test_f32_keys_sorted_windows_search(m, kind, curves):
    d = 128
    if (d // curves) * m > 1024:
        pytest.skip("key wider than HC_MAX_KEY_BITS (the reference rejects it too)")
    n, nq = 3000, 48
    rows = float_rows(n, d, 1)
    qs = float_rows(nq, d, 2)
    qs[:4] = rows[[0, 5, 17, 2999]]  # self queries
    gi = H.MulticurvesIndex(rows, H.default_scheme(d, curves, m, kind))
    assert gi.dtype == "f32"
    oi = _oracle(rows, curves, m, kind)
    for c in range(curves):
        gk = gi.keys(rows[:200], c)
        w = gk.shape[1]
        ok = np.stack([oi.query_key(rows[i], c)[:w] for i in range(200)])
        np.testing.assert_array_equal(gk, ok)
        gids, gkeys = gi.subindex(c, with_keys=True)
        okeys, oids = oi.sorted(c)
        np.testing.assert_array_equal(gids, oids)
        np.testing.assert_array_equal(gkeys, okeys)
    for depth in (1, 7, 64, 350):
        r, b, e = gi.windows(qs, depth)
        orr, ob, oe = oi.windows(qs, depth)
        np.testing.assert_array_equal(r, orr)
        np.testing.assert_array_equal(b, ob)
        np.testing.assert_array_equal(e, oe)
        cands = gi.candidates(qs[:16], depth)
        for q in range(16):
            np.testing.assert_array_equal(cands[q], oi.candidates(qs[q], depth))
        _check_search(gi, oi, qs, 10, depth)


@pytest.mark.parametrize("k", [1, 10, 33, 100, 256])
def test_f32_k_sweep(k):
    rows = float_rows(4000, 128, 3)
    qs = float_rows(64, 128, 4)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16))
    oi = _oracle(rows, 8, 16, H.HILBERT)
    _check_search(gi, oi, qs, k, 200)


@pytest.mark.parametrize("d,curves", [(128, 8), (96, 6), (64, 4), (20, 3), (1, 1)])
def test_f32_integer_components_bit_exact(d, curves):
    """Integer-valued components: every term and partial sum is exact, so the
    tree order cannot matter -- distances are bit-identical, ties by id."""
    rng = np.random.default_rng(5)
    rows = rng.integers(-60, 61, size=(2500, d)).astype(np.float32)
    rows[100:140] = rows[7]
    qs = rng.integers(-60, 61, size=(40, d)).astype(np.float32)
    qs[0] = rows[7]
    gi = H.MulticurvesIndex(rows, H.default_scheme(d, curves, 16))
    oi = _oracle(rows, curves, 16, H.HILBERT)
    for depth in (5, 300):
        _check_search(gi, oi, qs, 50, depth, exact=True)
    # brute force: exact kNN through the pair top-k
    ids, sq, ln = gi.brute_force(qs, 50)
    oids, odist, oln = P.brute_force(rows, qs, 50)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(ids, oids)
    assert gi.rooted(sq).tobytes() == odist.tobytes()


@pytest.mark.parametrize("k", [1, 16, 100])
def test_f32_brute_force(k):
    rows = float_rows(70000, 128, 6)  # > one 32768-row brute-force chunk
    qs = float_rows(20, 128, 7)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16))
    ids, sq, ln = gi.brute_force(qs, k)
    oids, odist, oln = P.brute_force(rows, qs, k)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(ids, oids)
    assert gi.rooted(sq).tobytes() == odist.tobytes()


def test_f32_small_batch_paths_and_device_buffers():
    """nq = 1 .. 300 runs the CTA-per-query gather; torch CUDA in/out == host."""
    import torch
    rows = float_rows(5000, 128, 8)
    qs = float_rows(300, 128, 9)
    gi = H.MulticurvesIndex(torch.from_numpy(rows).cuda(), H.default_scheme(128, 8, 16))
    oi = _oracle(rows, 8, 16, H.HILBERT)
    for nq in (1, 3, 64, 300):
        _check_search(gi, oi, qs[:nq], 10, 350)
    ids, sq, ln = gi.search_batch(torch.from_numpy(qs).cuda(), 10, 350)
    hids, hsq, hln = gi.search_batch(qs, 10, 350)
    np.testing.assert_array_equal(ids.cpu().numpy(), hids)
    assert sq.dtype == torch.float64
    assert sq.cpu().numpy().tobytes() == hsq.tobytes()
    np.testing.assert_array_equal(ln.cpu().numpy(), hln)


def test_f32_large_candidate_sets():
    """C x depth beyond the register union (shared-memory and global-table unions)."""
    rows = float_rows(30000, 128, 10)
    qs = float_rows(8, 128, 11)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 16, 8))
    oi = _oracle(rows, 16, 8, H.HILBERT)
    for depth in (700, 3000):
        _check_search(gi, oi, qs, 20, depth)


def test_f32_insert_save_load(tmp_path):
    rows = float_rows(6000, 128, 12)
    qs = float_rows(32, 128, 13)
    scheme = H.default_scheme(128, 8, 16)
    full = H.MulticurvesIndex(rows, scheme)
    grown = H.MulticurvesIndex(rows[:2500], scheme)
    grown.insert(rows[2500:4000])
    grown.insert(rows[4000:])
    for c in range(8):
        np.testing.assert_array_equal(grown.subindex(c), full.subindex(c))
    a = full.search_batch(qs, 10, 100)
    b = grown.search_batch(qs, 10, 100)
    for x, y in zip(a, b):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()
    path = str(tmp_path / "f32.hcg")
    full.save(path)
    back = H.MulticurvesIndex.load(path, scheme, H.RAW)
    assert back.dtype == "f32"
    c = back.search_batch(qs, 10, 100)
    for x, y in zip(a, c):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()


def test_f32_fvecs_to_index(tmp_path):
    """fvecs (vecio.cpp:18-61) -> float rows -> index, no byte view involved."""
    rows = float_rows(1000, 128, 14)
    path = str(tmp_path / "base.fvecs")
    H.write_vectors(path, rows, "fvecs")
    back = H.read_vectors(path, "fvecs", dtype="f32")
    assert back.tobytes() == rows.tobytes()
    gi = H.MulticurvesIndex(back, H.default_scheme(128, 8, 16))
    oi = _oracle(rows, 8, 16, H.HILBERT)
    _check_search(gi, oi, rows[:16], 5, 64)


def test_f32_errors():
    rows = float_rows(500, 128, 15)
    scheme = H.default_scheme(128, 8, 16)
    bad = rows.copy()
    bad[123, 45] = np.nan
    with pytest.raises(HcgError) as e:
        H.MulticurvesIndex(bad, scheme)
    assert e.value.code == -3  # HCG_ENONFINITE (curve.cpp:167)
    bad[123, 45] = np.inf
    with pytest.raises(HcgError):
        H.MulticurvesIndex(bad, scheme)
    gi = H.MulticurvesIndex(rows, scheme)
    q = rows[:4].copy()
    q[2, 0] = -np.inf
    with pytest.raises(HcgError) as e:
        gi.search_batch(q, 5, 10)
    assert e.value.code == -3
    with pytest.raises(HcgError):
        gi.windows(q, 10)
    with pytest.raises(HcgError):
        gi.insert(bad[:200])
    assert gi.size() == 500
    # u8 queries against an f32 index (and the packed / timed u8-only calls)
    with pytest.raises(HcgError):
        gi.search_batch(np.zeros((2, 128), np.uint8), 5, 10)
    with pytest.raises(HcgError):
        gi.search_packed(rows[:2], 5, 10)
    # 129 float components exceed the 512-byte row
    with pytest.raises(HcgError):
        H.MulticurvesIndex(float_rows(10, 129, 0), H.default_scheme(129, 3, 8))


def test_f32_large_batch():
    """Warp-per-query f32 gather with the curve-0 batch order (>= 16K queries)."""
    rows = float_rows(20_000, 128, 21)
    qs = float_rows(17_000, 128, 22)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16))
    oi = _oracle(rows, 8, 16, H.HILBERT)
    _check_search(gi, oi, qs, 10, 300)


def test_f32_sequential_sum_near_ties():
    """Rows whose squared distances depend on the summation order: with
    (2^27, 1, 1, ...) against a zero query, the reference's sequential sum
    (vecio.cpp:90-93) absorbs every 1 into 2^54 (ulp 4), so the row ties
    with (2^27, 0, 0, ...) and the lower id wins; any other order (e.g. a
    tree) would add the ones up and put it second."""
    d = 128
    rng = np.random.default_rng(11)
    rows = (rng.standard_normal((300, d)) * 5e7).astype(np.float32)  # far: d^2 ~ 3e17 > 2^54
    crafted = np.zeros((4, d), np.float32)
    crafted[:, 0] = np.float32(2.0 ** 27)
    crafted[0, 1:] = 1.0       # id 100: sequential sum 2^54
    crafted[1, 1:] = 0.0       # id 101: 2^54 exactly
    crafted[2, 1:5] = 3.0      # id 102: 2^54 + 9 + ... rounds
    crafted[3, 1:] = -1.0      # id 103: same as 100
    rows[100:104] = crafted
    q = np.zeros((1, d), np.float32)
    scheme = H.default_scheme(d, 1, 8)
    gi = H.MulticurvesIndex(rows, scheme)
    oi = P.Oracle(rows, 1, 8, H.HILBERT)
    for fn in ("search", "brute"):
        if fn == "search":
            ids, sq, ln = gi.search_batch(q, 8, 1000)
            oids, odist, oln = oi.search(q, 8, 1000)
        else:
            ids, sq, ln = gi.brute_force(q, 8)
            oids, odist, oln = P.brute_force(rows, q, 8)
        np.testing.assert_array_equal(ids, oids)
        assert gi.rooted(sq).tobytes() == odist.tobytes()
    ids, sq, _ = gi.brute_force(q, 8)
    pos = {int(i): r for r, i in enumerate(ids[0])}
    assert sq[0, pos[100]] == sq[0, pos[101]] == 2.0 ** 54  # the ones were absorbed
    assert pos[100] < pos[101] < pos[103]
