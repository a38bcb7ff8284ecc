"""K5 on the tensor cores (csrc/brute_tc.cu): exact kNN ground truth via
tcgen05.mma kind::i8 (u8 x u8 -> s32) against the oracle's brute_force_knn
(vecio.cpp:115-122) -- bit-exact ids, distances and (distance, id) tie order.

The tensor-core path serves u8 rows of 128 bytes with k <= 32; other shapes
use the CUDA-core K5 (covered in test_gpu_parity.py)."""
import numpy as np
import pytest

from oracle import pyoracle as P
from hcg_testutil import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_1209_0410_b200 as H  # noqa: E402


def _check(gi, rows, qs, k, view=H.RAW):
    ids, sq, ln = gi.brute_force(qs, k)
    bids, bdist, bln = P.brute_force(view.floats(rows), view.floats(qs), k, ids=None)
    np.testing.assert_array_equal(ln, bln)
    d = gi.rooted(sq)
    for q in range(qs.shape[0]):
        L = int(ln[q])  # past the list: id 2^64-1 here, 0 in the oracle
        np.testing.assert_array_equal(ids[q, :L], bids[q, :L])
        assert d[q, :L].tobytes() == bdist[q, :L].tobytes()
        assert (ids[q, L:] == np.uint64(2**64 - 1)).all()


@pytest.mark.parametrize("k", [1, 8, 10, 16, 17, 32])
def test_tc_brute_matches_oracle(k):
    # n not a multiple of the 256-row tile, nq not a multiple of the 128-query tile
    rows = P.gen_rows(0, 41_234)
    qs = P.gen_queries(0, 300, 41_234)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    _check(gi, rows, qs, k, H.LIFTED)


def test_tc_brute_extremes_and_ties():
    """All-255 / all-0 rows (largest q.x and S), duplicated rows (ties by id),
    a query equal to a row (S = 0)."""
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 256, size=(5000, 128), dtype=np.uint8)
    rows[0] = 255
    rows[1] = 0
    rows[100:140] = rows[7]
    rows[4999] = rows[7]
    qs = rng.integers(0, 256, size=(130, 128), dtype=np.uint8)
    qs[0] = 255
    qs[1] = 0
    qs[2] = rows[7]
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 8), H.RAW)
    for k in (1, 5, 32):
        _check(gi, rows, qs, k)


def test_tc_brute_many_chunks_and_tiny_inputs():
    rows = P.gen_rows(0, 300_000)
    qs = P.gen_queries(0, 20, 300_000)
    gi = H.MulticurvesIndex(rows, H.default_scheme(128, 8, 16), H.LIFTED)
    _check(gi, rows, qs, 10, H.LIFTED)
    # fewer rows than one tile, one query, k > n
    small = rows[:7]
    gs = H.MulticurvesIndex(small, H.default_scheme(128, 8, 16), H.LIFTED)
    _check(gs, small, qs[:1], 10, H.LIFTED)


def test_tc_brute_sharded_ids():
    """Affine ids (shard r of G: id = r + slot * G) survive the tensor-core path."""
    rows = P.gen_rows(0, 9000)
    qs = P.gen_queries(0, 50, 9000)
    G = 3
    for r in range(G):
        sel = rows[r::G]
        gi = H.MulticurvesIndex(sel, H.default_scheme(128, 8, 16), H.LIFTED, id_base=r, id_stride=G)
        ids, sq, ln = gi.brute_force(qs, 10)
        bids, bdist, bln = P.brute_force(H.LIFTED.floats(sel), H.LIFTED.floats(qs), 10,
                                         ids=np.arange(r, 9000, G, dtype=np.uint64))
        np.testing.assert_array_equal(ids, bids)
        assert gi.rooted(sq).tobytes() == bdist.tobytes()
