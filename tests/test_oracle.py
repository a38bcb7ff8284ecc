"""The CPU oracle, pinned: SURVEY.md §A golden vectors (produced by the shipped
reference code), the committed reference fixture (tests/golden/ref_fixture.npz,
made by running the reference TUs), SPEC.md's per-op examples, and -- where the
reference tree was present at build time -- a live cross-check against the
reference TUs themselves (oracle/_ref)."""
import ctypes
import os
from fractions import Fraction
from math import comb

import numpy as np
import pytest

from oracle import pyoracle as P

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = np.load(os.path.join(HERE, "golden", "ref_fixture.npz"))
R16 = [0, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 17, 99, 128]


def key16(kind, vals, m, view):
    f = P.view_floats(np.array(vals, np.uint8), view)
    return P.key_hex(P.curve_encode(kind, [P.quantize(float(x), m) for x in f], m))


# ------------------------------------------------------------ SURVEY §A ----
def test_quantizer_raw_m8_six_cells():
    """bytes collapse to 6 cells at m=8 (curve.cpp:166-174)."""
    table = {0: 0x80, 1: 0xBF}
    table.update({b: 0xC0 for b in range(2, 8)})
    table.update({b: 0xC1 for b in range(8, 32)})
    table.update({b: 0xC2 for b in range(32, 128)})
    table.update({b: 0xC3 for b in range(128, 256)})
    for b in range(256):
        assert P.quantize(float(b), 8) == table[b]


def test_distinct_cells_per_m():
    for m, want in ((8, 6), (12, 48), (16, 256), (20, 256), (24, 256), (32, 256)):
        assert len({P.quantize(float(b), m) for b in range(256)}) == want


def test_lifted_view_cells():
    f = P.view_floats(np.arange(256, dtype=np.uint8), P.LIFTED)
    for b in range(256):
        assert P.quantize(float(f[b]), 17) == (0x17F00 | b)
        assert P.quantize(float(f[b]), 16) == (0xBF80 | (b >> 1))


def test_float_to_ordinal_goldens():
    o = P.orc().orc_float_to_ordinal
    assert o(0.0) == 0x80000000
    assert o(-0.0) == 0x7FFFFFFF
    assert o(1.0) == 0xBF800000
    assert o(255.0) == 0xC37F0000
    chain = [-1.5, -0.25, 0.0, 0.25, 1.5]
    assert [o(x) for x in chain] == sorted(o(x) for x in chain)


def test_nonfinite_and_capacity_rejected():
    v = ctypes.c_uint64()
    assert P.orc().orc_quantize(ctypes.c_float(float("nan")), 8, ctypes.byref(v)) != 0
    assert P.orc().orc_quantize(ctypes.c_float(float("inf")), 8, ctypes.byref(v)) != 0
    with pytest.raises(ValueError):
        P.curve_encode(P.HILBERT, [0] * 17, 64)  # 1088 bits > 1024


def test_curve_small_goldens():
    # Hilbert d=2, m=1: key 0->(0,0), 1->(0,1), 2->(1,1), 3->(1,0)
    for key, pt in enumerate([(0, 0), (0, 1), (1, 1), (1, 0)]):
        assert int(P.curve_encode(P.HILBERT, pt, 1)[0]) == key
    assert int(P.curve_encode(P.ZORDER, (1, 1), 1)[0]) == 3
    assert int(P.curve_encode(P.ZORDER, (0, 0), 1)[0]) == 0


@pytest.mark.parametrize("view,m,kind,vals,want", [
    (P.RAW, 8, P.ZORDER, [0] * 16, "ffff0000000000000000000000000000"),
    (P.RAW, 8, P.HILBERT, [0] * 16, "aaaa0000000000000000000000000000"),
    (P.RAW, 8, P.ZORDER, [255] * 16, "ffffffff0000000000000000ffffffff"),
    (P.RAW, 8, P.HILBERT, [255] * 16, "aaaaaaaa0000000000000000aaaaaaaa"),
    (P.RAW, 8, P.ZORDER, R16, "ffff3fff400040004000400040fb471d"),
    (P.RAW, 8, P.HILBERT, R16, "aaaa2aaaffffffffffffffff200aefde"),
    (P.RAW, 16, P.ZORDER, R16, "ffff3fff400040004000400040fb471d4926124a0928027001cc004200220008"),
    (P.RAW, 16, P.HILBERT, R16, "aaaa2aaaffffffffffffffff200aefde37f079c132e4e29039511d16f56a0d69"),
    (P.LIFTED, 16, P.ZORDER, R16, "ffff0000ffffffffffffffffffffffffffff0019002a00ca017406280b4030c2"),
    (P.LIFTED, 16, P.HILBERT, R16, "aaaa0000aaaaaaaaaaaaaaaaaaaaaaaaaaaafff77ffbbfe89ff18fda77e85843"),
    (P.LIFTED, 16, P.HILBERT, [0] * 16, "aaaa0000aaaaaaaaaaaaaaaaaaaaaaaaaaaa0000000000000000000000000000"),
])
def test_16d_key_goldens(view, m, kind, vals, want):
    """16-d keys printed by the shipped reference (ExtendedKey::to_hex)."""
    assert key16(kind, vals, m, view) == want


def test_select_top_k_golden():
    """select_top_k(k=4) on {(7,4),(3,4),(9,1),(5,4),(1,9),(2,0)} -> (2,0),(9,1),(3,2),(5,2)."""
    # restate through brute_force: 1-d points whose squared distance to 0 are the given values
    sq = {7: 4, 3: 4, 9: 1, 5: 4, 1: 9, 2: 0}
    pts = np.array([[np.sqrt(v)] for v in sq.values()], np.float32)
    idv = np.array(list(sq.keys()), np.uint64)
    oi, od, ln = P.brute_force(pts, np.zeros((1, 1), np.float32), 4, ids=idv)
    assert list(oi[0]) == [2, 9, 3, 5]
    assert list(od[0]) == [0.0, 1.0, 2.0, 2.0]
    if P.ref_available():
        out_i = np.zeros(4, np.uint64)
        out_d = np.zeros(4, np.float64)
        n = P.ref().ref_select_top_k(idv, np.array(list(sq.values()), np.float64), 6, 4, out_i, out_d)
        assert n == 4 and list(out_i) == [2, 9, 3, 5] and list(out_d) == [0.0, 1.0, 2.0, 2.0]


def test_euclidean_3_4_5():
    oi, od, _ = P.brute_force(np.array([[3.0, 4.0]], np.float32), np.zeros((1, 2), np.float32), 1)
    assert od[0, 0] == 5.0


# ------------------------------------------------ SPEC curve properties ----
@pytest.mark.parametrize("kind", [P.ZORDER, P.HILBERT])
def test_roundtrip_d2_m8_exhaustive(kind):
    """SPEC.md:50,68 (Acceptance 1): decode(encode(p)) == p over the full d=2, m=8 grid."""
    seen = set()
    for x in range(0, 256, 3):
        for y in range(256):
            key = P.curve_encode(kind, (x, y), 8)
            assert tuple(int(c) for c in P.curve_decode(kind, key, 2, 8)) == (x, y)
            seen.add(int(key[0]))
    assert len(seen) == len(range(0, 256, 3)) * 256


def test_hilbert_adjacency_and_bijection():
    """unit-step adjacency (d=2, m=4) and bijection (d=3, m=3)."""
    cells = [tuple(int(c) for c in P.curve_decode(P.HILBERT, [k], 2, 4)) for k in range(256)]
    assert len(set(cells)) == 256
    for a, b in zip(cells, cells[1:]):
        assert sum(abs(i - j) for i, j in zip(a, b)) == 1
    keys = {int(P.curve_encode(P.HILBERT, (x, y, z), 3)[0])
            for x in range(8) for y in range(8) for z in range(8)}
    assert keys == set(range(512))


# --------------------------------------------- reference fixture (pins) ----
@pytest.mark.parametrize("view", [P.RAW, P.LIFTED])
def test_fixture_quantizer(view):
    f = P.view_floats(np.arange(256, dtype=np.uint8), view)
    for m in (8, 12, 16, 17, 20, 24, 32):
        got = np.array([P.quantize(float(x), m) for x in f], np.uint64)
        np.testing.assert_array_equal(got, FIX[f"quant_v{view}_m{m}"])


def test_fixture_curve_keys():
    for kind in (P.ZORDER, P.HILBERT):
        for d, m in ((2, 8), (3, 5), (16, 8), (16, 16), (8, 32), (128, 8), (64, 16)):
            pts = FIX[f"pts_k{kind}_d{d}_m{m}"]
            want = FIX[f"keys_k{kind}_d{d}_m{m}"]
            for i in range(len(pts)):
                np.testing.assert_array_equal(P.curve_encode(kind, pts[i], m), want[i])


def test_fixture_generator():
    """The §8(d) generator restated in the oracle produces the fixture's bytes."""
    n = FIX["rows"].shape[0]
    np.testing.assert_array_equal(P.gen_rows(0, n), FIX["rows"])
    q = P.gen_queries(0, FIX["queries"].shape[0], n)
    q[0] = FIX["rows"][123]
    np.testing.assert_array_equal(q, FIX["queries"])


@pytest.mark.parametrize("view,m", [(P.RAW, 8), (P.LIFTED, 16)])
@pytest.mark.parametrize("kind", [P.HILBERT, P.ZORDER])
def test_fixture_index_and_search(view, m, kind):
    rows, qs = FIX["rows"], FIX["queries"]
    tag = f"v{view}_k{kind}"
    oi = P.Oracle(P.view_floats(rows, view), 8, m, kind)
    for c in (0, 3, 7):
        keys, ids = oi.sorted(c)
        np.testing.assert_array_equal(ids, FIX[f"sorted_ids_{tag}_c{c}"])
        np.testing.assert_array_equal(keys, FIX[f"sorted_keys_{tag}_c{c}"])
    qf = P.view_floats(qs, view)
    for depth in (1, 7, 64, 350, 5000):
        r, b, e = oi.windows(qf, depth)
        np.testing.assert_array_equal(np.stack([r, b, e]), FIX[f"win_{tag}_d{depth}"])
    for depth in (7, 350):
        np.testing.assert_array_equal(oi.candidates(qf[5], depth), FIX[f"cand_{tag}_d{depth}_q5"])
    for k, depth in ((10, 64), (10, 350), (100, 350), (1, 1)):
        ids, dist, ln = oi.search(qf, k, depth)
        np.testing.assert_array_equal(ln, FIX[f"searchl_{tag}_k{k}_d{depth}"])
        np.testing.assert_array_equal(ids, FIX[f"search_{tag}_k{k}_d{depth}"])
        assert dist.tobytes() == FIX[f"searchd_{tag}_k{k}_d{depth}"].tobytes()
    if kind == P.HILBERT:
        ids, dist, _ = P.brute_force(P.view_floats(rows, view), qf, 10)
        np.testing.assert_array_equal(ids, FIX[f"brute_v{view}"])
        assert dist.tobytes() == FIX[f"bruted_v{view}"].tobytes()


# ------------------------------------------------------- SPEC examples ----
def test_window_edges_and_depth_ge_n():
    """depth >= n -> all ids; a query key below every key ->
    the first depth entries (boundary spill)."""
    rows = P.gen_rows(0, 300)
    oi = P.Oracle(P.view_floats(rows, P.RAW), 4, 8)
    q = P.view_floats(rows[:1], P.RAW)
    assert len(oi.candidates(q[0], 1000)) == 300
    low = np.zeros((1, 128), np.float32) - 1.0  # quantizes below every stored key
    r, b, e = oi.windows(low, 10)
    assert (r == 0).all() and (b == 0).all() and (e == 10).all()
    high = np.full((1, 128), 1e30, np.float32)  # the max cell is the max key on the Z-order curve
    r, b, e = P.Oracle(P.view_floats(rows, P.RAW), 4, 8, P.ZORDER).windows(high, 10)
    assert (r == 300).all() and (b == 290).all() and (e == 300).all()


def test_self_query_and_one_curve_is_brute_force():
    """SPEC.md:251-252."""
    rows = P.gen_rows(0, 1500)
    f = P.view_floats(rows, P.RAW)
    oi = P.Oracle(f, 8, 8)
    ids, dist, _ = oi.search(f[[0, 10, 700]], 1, 1)
    assert (dist[:, 0] == 0).all()
    one = P.Oracle(f, 1, 8)
    qs = P.view_floats(P.gen_queries(0, 12, 1500), P.RAW)
    a = one.search(qs, 10, 1500)
    b = P.brute_force(f, qs, 10)
    np.testing.assert_array_equal(a[0], b[0])
    assert a[1].tobytes() == b[1].tobytes()


def test_recall_monotone_in_depth():
    """candidate sets are nested in depth, so recall is monotone."""
    rows = P.gen_rows(0, 4000)
    f = P.view_floats(rows, P.LIFTED)
    qs = P.view_floats(P.gen_queries(0, 30, 4000), P.LIFTED)
    oi = P.Oracle(f, 8, 16)
    truth = P.brute_force(f, qs, 10)[0]
    prev = -1.0
    for depth in (8, 32, 128, 512):
        got = oi.search(qs, 10, depth)[0]
        rec = np.mean([len(set(a) & set(b)) / 10 for a, b in zip(got, truth)])
        assert rec >= prev
        prev = rec
        c_small = set(oi.candidates(qs[0], depth).tolist())
        c_big = set(oi.candidates(qs[0], depth * 2).tolist())
        assert c_small <= c_big


def test_sharded_oracle_full_depth_at_least_as_good():
    """SURVEY F7 / PAPER.md:844-846: with per-shard depth = sequential depth the
    sharded candidate union contains the sequential one, so every sharded
    result distance is <= the sequential one at the same rank."""
    rows = P.gen_rows(0, 3000)
    f = P.view_floats(rows, P.LIFTED)
    qs = P.view_floats(P.gen_queries(0, 20, 3000), P.LIFTED)
    seq = P.Oracle(f, 8, 16).search(qs, 10, 64)
    sh = P.sharded_search(f, qs, 4, 8, 16, 10, 64)
    assert (sh[1] <= seq[1] + 0.0).all()


# ----------------------------------------- live cross-check vs reference ----
@pytest.mark.skipif(not P.ref_available(), reason="oracle/_ref not built (reference tree absent)")
@pytest.mark.parametrize("view,m", [(P.RAW, 8), (P.LIFTED, 16)])
@pytest.mark.parametrize("curves", [1, 2, 4, 8, 16])
def test_oracle_equals_reference_tus(view, m, curves):
    if (128 // curves) * m > 1024:
        pytest.skip("key wider than HC_MAX_KEY_BITS")
    rows = P.gen_rows(5, 1200)
    qs = P.gen_queries(3, 16, 1200)
    ri = P.RefIndex(rows, curves, m, P.HILBERT, view)
    oi = P.Oracle(P.view_floats(rows, view), curves, m, P.HILBERT)
    for c in range(curves):
        okeys, oids = oi.sorted(c)
        rkeys, rids = ri.sorted(c, okeys.shape[1])
        np.testing.assert_array_equal(oids, rids)
        np.testing.assert_array_equal(okeys, rkeys)
    for depth in (3, 100):
        a = oi.search(P.view_floats(qs, view), 10, depth)
        b = ri.search(qs, 10, depth, threads=1)
        np.testing.assert_array_equal(a[0], b[0])
        assert a[1].tobytes() == b[1].tobytes()


# ------------------------------------------------- equivalence planner ----
def _tail_exact(trials, p, phi):
    return sum(comb(trials, k) * p**k * (1 - p)**(trials - k) for k in range(phi + 1, trials + 1))


def test_planner_binomial_tail_exact():
    """exact rational arithmetic for Phi <= 64."""
    import paper_1209_0410_b200 as H
    assert H.binomial_tail(10, 0.3, 10) == 0.0
    assert abs(H.binomial_tail(1, 0.5, 0) - 0.5) < 1e-15
    for trials in (8, 32, 64):
        for ell in (2, 4, 8):
            p = Fraction(1, ell)
            for phi in range(0, trials, 7):
                exact = float(_tail_exact(trials, p, phi))
                got = H.binomial_tail(trials, 1.0 / ell, phi)
                assert abs(got - exact) <= 1e-12 + 1e-9 * exact


def test_planner_bound_and_plan():
    import paper_1209_0410_b200 as H
    assert H.miss_bound(64, 1, 64) == 0.0
    assert H.miss_bound(64, 4, 64) == 0.0
    prev = 1.0
    for phi in range(0, 129):
        b = H.miss_bound(128, 8, phi)
        assert b <= prev + 1e-15
        prev = b
    # SURVEY §8(d) config 3 table (re-derived by the planner)
    assert [H.shard_probe_depth(350, g) for g in (2, 4, 8)] == [226, 134, 80]
    assert [H.shard_probe_depth(256, g) for g in (2, 4, 8)] == [170, 102, 64]


def test_planner_monte_carlo_validates_bound():
    """the empirical miss frequency stays under the bound."""
    import paper_1209_0410_b200 as H
    rng = np.random.default_rng(0)
    Phi, ell = 128, 8
    phi = H.plan_depth(Phi, ell, 0.02)
    trials = 20000
    a = rng.multinomial(Phi, [1 / ell] * ell, size=trials)
    b = rng.multinomial(Phi, [1 / ell] * ell, size=trials)
    miss = np.mean((a.max(axis=1) > phi) | (b.max(axis=1) > phi))
    sigma = np.sqrt(0.02 * 0.98 / trials)
    assert miss <= H.miss_bound(Phi, ell, phi) + 3 * sigma
