"""Incremental insert and persistence on the B200 (multicurves.hpp:79,96-98;
SPEC.md:227-235,268): build(A) + insert(B) equals build(A u B) entry for entry
(SPEC's order-independence oracle), including the case where B moves a
curve's common key prefix (rebuild path); save -> load round-trips bit-exactly."""
import numpy as np
import pytest

from hcg_testutil import gpu_available
from oracle import pyoracle as P

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402


def _same_index(a, b, qs, curves, k=10, depth=200):
    for c in range(curves):
        ia, ka = a.subindex(c, with_keys=True)
        ib, kb = b.subindex(c, with_keys=True)
        np.testing.assert_array_equal(ia, ib)
        np.testing.assert_array_equal(ka, kb)
    ra = a.search_batch(qs, k, depth)
    rb = b.search_batch(qs, k, depth)
    for x, y in zip(ra, rb):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("view,m", [(H.RAW, 8), (H.LIFTED, 16)])
def test_insert_equals_build_of_union(view, m):
    rows = P.gen_rows(0, 6000)
    qs = P.gen_queries(0, 40, 6000)
    sch = H.default_scheme(128, 8, m)
    full = H.MulticurvesIndex(rows, sch, view)
    inc = H.MulticurvesIndex(rows[:4000], sch, view)
    inc.insert(rows[4000:4001])          # single row (the reference's per-vector insert)
    inc.insert(rows[4001:5500])
    inc.insert(rows[5500:])
    assert inc.size() == 6000
    _same_index(inc, full, qs, 8)
    oi = P.Oracle(view.floats(rows), 8, m)
    ids, dist, ln = oi.search(view.floats(qs), 10, 200)
    gi, gs, gl = inc.search_batch(qs, 10, 200)
    np.testing.assert_array_equal(gi, ids)


def test_insert_that_moves_the_common_prefix():
    rng = np.random.default_rng(3)
    low = rng.integers(0, 40, (3000, 128), dtype=np.uint8)
    high = rng.integers(200, 256, (500, 128), dtype=np.uint8)
    both = np.concatenate([low, high])
    qs = np.concatenate([low[:10], high[:10]])
    sch = H.default_scheme(128, 8, 16)
    inc = H.MulticurvesIndex(low, sch, H.LIFTED)
    inc.insert(high)
    _same_index(inc, H.MulticurvesIndex(both, sch, H.LIFTED), qs, 8)


def test_insert_into_empty_index_equals_build():
    rows = P.gen_rows(0, 100)
    sch = H.default_scheme(128, 4, 8)
    e = H.MulticurvesIndex(rows[:0], sch, H.RAW)
    e.insert(rows)
    _same_index(e, H.MulticurvesIndex(rows, sch, H.RAW), rows[:5], 4)


@pytest.mark.parametrize("view,m,kind", [(H.RAW, 8, H.HILBERT), (H.LIFTED, 16, H.ZORDER)])
def test_save_load_round_trip(tmp_path, view, m, kind):
    rows = np.random.default_rng(4).integers(0, 256, (5000, 100), dtype=np.uint8)
    qs = rows[:30]
    sch = H.default_scheme(100, 7, m, kind)
    a = H.MulticurvesIndex(rows, sch, view)
    path = str(tmp_path / "idx.hcg")
    a.save(path)
    b = H.MulticurvesIndex.load(path, sch, view)
    assert b.size() == 5000 and b.curves() == 7
    _same_index(a, b, qs, 7)
    b.save(str(tmp_path / "again.hcg"))
    assert open(path, "rb").read() == open(str(tmp_path / "again.hcg"), "rb").read()


def test_load_rejects_garbage(tmp_path):
    p = tmp_path / "bad.hcg"
    p.write_bytes(b"not an index at all")
    with pytest.raises(H.HcgIOError):
        H.MulticurvesIndex.load(str(p), H.default_scheme(128, 8), H.RAW)


def test_load_recovers_scheme_and_view(tmp_path):
    """hcg_describe: a saved index loads without the caller restating its
    scheme or view (multicurves.hpp:98 takes only the path)."""
    import paper_1209_0410_b200 as H
    from oracle import pyoracle as P
    rows = P.gen_rows(0, 3000)
    qs = P.gen_queries(0, 20, 3000)
    scheme = H.default_scheme(128, 8, 16)
    gi = H.MulticurvesIndex(rows, scheme, H.LIFTED)
    path = str(tmp_path / "x.hcg")
    gi.save(path)
    back = H.MulticurvesIndex.load(path)
    assert back.scheme.assignment == scheme.assignment and back.scheme.bits_per_dim == 16
    assert back.view.offset == 1.0 and back.view.scale == 1.0 / 256
    a, b = gi.search_batch(qs, 10, 100), back.search_batch(qs, 10, 100)
    for x, y in zip(a, b):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()
    assert gi.search(qs[0], H.SearchParams(10, 100)) == back.search(qs[0], H.SearchParams(10, 100))
    np.testing.assert_array_equal(back.retrieve_candidates(qs[3], 2, 50), gi.subindex(2)[
        int(gi.windows(qs[3], 50)[1][0, 2]):int(gi.windows(qs[3], 50)[2][0, 2])])


@pytest.mark.parametrize("view,m", [(H.LIFTED, 16), (H.RAW, 8)])
def test_insert_then_large_batch_search(view, m):
    """An inserted index searched with >= 16K queries runs the union-less
    k_gather_nu, which maps physical rows back to ids through the id table
    that inserts extend (appended rows sit at physical = id slot): results
    equal the oracle over all rows and a fresh build of the union."""
    rows = P.gen_rows(0, 9000)
    qs = P.gen_queries(0, 20000, 9000)
    sch = H.default_scheme(128, 8, m)
    inc = H.MulticurvesIndex(rows[:6000], sch, view)
    inc.insert(rows[6000:7500])
    inc.insert(rows[7500:])
    full = H.MulticurvesIndex(rows, sch, view)
    for k, depth in ((10, 350), (1, 40), (32, 1000)):
        gi, gs, gl = inc.search_batch(qs, k, depth)
        fi, fs, fl = full.search_batch(qs, k, depth)
        np.testing.assert_array_equal(gi, fi)
        np.testing.assert_array_equal(gs, fs)
        np.testing.assert_array_equal(gl, fl)
    oi = P.Oracle(view.floats(rows), 8, m)
    oids, odist, oln = oi.search(view.floats(qs), 10, 350)
    gi, gs, gl = inc.search_batch(qs, 10, 350)
    np.testing.assert_array_equal(gl, oln)
    np.testing.assert_array_equal(gi, oids)
    assert inc.rooted(gs).tobytes() == odist.tobytes()


@pytest.mark.parametrize("how", ["out_of_range", "duplicate"])
def test_load_rejects_corrupt_slots(tmp_path, how):
    """A slot array that is not a permutation of the rows fails with
    HCG_EIO instead of becoming out-of-bounds row gathers."""
    rows = P.gen_rows(0, 2000)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 4, 8), H.RAW)
    path = tmp_path / "x.hcg"
    gi.save(str(path))
    raw = bytearray(path.read_bytes())
    # the last curve's slots are the 2000 u32 right before the 8-byte trailer
    end = len(raw) - 8
    slots = np.frombuffer(bytes(raw[end - 4 * 2000:end]), np.uint32).copy()
    if how == "out_of_range":
        slots[17] = 2000
    else:
        slots[17] = slots[18]
    raw[end - 4 * 2000:end] = slots.tobytes()
    path.write_bytes(bytes(raw))
    with pytest.raises(H.HcgIOError):
        H.MulticurvesIndex.load(str(path))
