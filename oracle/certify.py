"""Certificate parity for configurations too large for a CPU index (test
infrastructure: only tests/, bench.py's checks and smoke() use it).

For a sample of queries, the answer of one shard (or a whole unsharded index)
is recomputed from the reference's semantics, trusting the GPU only for which
ids sit at the sorted positions around each window -- and checking those:

  * every id at positions [begin - 1, end] of curve c is regenerated from the
    counter-based generator and keyed by the oracle
    (curve.cpp:62-174 restated in hc_oracle.cpp); the entries must be in
    (key, id) order (multicurves.hpp:47-48);
  * the GPU's rank must be the lower bound of the oracle's query key
    (key(rank - 1) < qkey <= key(rank), multicurves.hpp:57-58);
  * the window must follow the header rule from (rank, depth, n)
    (multicurves.hpp:60-63);
  * the candidate union of the windows is scored with exact squared distances
    of the view floats (vecio.cpp:87-95: every term and partial sum is exact
    for the byte views) and the top-k taken by (distance, id)
    (vecio.cpp:101-113).

The per-shard lists are then merged by (distance, id) and
compared bit-for-bit with the GPU's merged result.  Cost is independent of the
index size: ~C x depth regenerated rows per query.
"""
from __future__ import annotations

import numpy as np

from . import pyoracle as P


def _key_int(words) -> int:
    v = 0
    for i, w in enumerate(words):
        v |= int(w) << (64 * i)
    return v


def window_rule(n: int, rank: int, depth: int):
    take = min(depth, n)
    begin = max(rank - take // 2, 0)
    if begin + take > n:
        begin = n - take
    return begin, begin + take


def certify_shard(index, qs_u8: np.ndarray, depth: int, k: int, view: int, m: int, kind: int = P.HILBERT):
    """Recompute one index's (shard's) top-k for every query of qs_u8 from
    reference semantics.  Returns (ids, dist, len, report); report counts the
    failed checks (all zero on a correct index)."""
    qs = np.ascontiguousarray(qs_u8, np.uint8)
    nq = qs.shape[0]
    n = index.size()
    C = index.curves()
    ranks, begins, ends = index.windows(qs, depth)
    oix = P.Oracle(P.view_floats(qs[:1], view), C, m, kind)
    W = [oix.words(c) for c in range(C)]
    bad = {"window_rule": 0, "sorted_neighbourhood": 0, "lower_bound": 0}
    ids_out = np.full((nq, k), np.uint64(2**64 - 1))
    dist_out = np.zeros((nq, k), np.float64)
    len_out = np.zeros(nq, np.uint32)
    qf_all = P.view_floats(qs, view).astype(np.float64)
    for q in range(nq):
        qf32 = P.view_floats(qs[q:q + 1], view)
        cand = []
        for c in range(C):
            r, b, e = int(ranks[q, c]), int(begins[q, c]), int(ends[q, c])
            if (b, e) != window_rule(n, r, depth):
                bad["window_rule"] += 1
            lo, hi = max(b - 1, 0), min(e + 1, n)
            ids = index.sorted_ids(c, lo, hi - lo)
            rows = P.gen_rows_ids(ids)
            keys = oix.keys(P.view_floats(rows, view), c)
            kint = [_key_int(keys[i, :W[c]]) for i in range(len(ids))]
            if any((kint[i], int(ids[i])) >= (kint[i + 1], int(ids[i + 1])) for i in range(len(ids) - 1)):
                bad["sorted_neighbourhood"] += 1
            qk = _key_int(oix.query_key(qf32[0], c)[:W[c]])
            if r - 1 >= lo and not kint[r - 1 - lo] < qk:
                bad["lower_bound"] += 1
            if r < hi and not qk <= kint[r - lo]:
                bad["lower_bound"] += 1
            if (r - 1 < lo and r > 0) or (r >= hi and r < n):
                bad["lower_bound"] += 1  # the rank must sit inside the fetched neighbourhood
            cand.append(ids[b - lo:e - lo])
        u = np.unique(np.concatenate(cand)) if cand else np.zeros(0, np.uint64)
        rows = P.view_floats(P.gen_rows_ids(u), view).astype(np.float64)
        d2 = ((rows - qf_all[q][None, :]) ** 2).sum(axis=1)  # exact: integer multiples of scale^2
        order = np.lexsort((u, d2))[:k]
        L = len(order)
        ids_out[q, :L] = u[order]
        dist_out[q, :L] = np.sqrt(d2[order])
        len_out[q] = L
    report = {"queries": nq, "curves": C, "rows": n, "depth": depth, "failed_checks": bad}
    return ids_out, dist_out, len_out, report
