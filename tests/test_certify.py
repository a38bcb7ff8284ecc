"""The certificate checker (oracle/certify.py) used for parity where a CPU
index of the whole configuration is infeasible (100M rows, N > 1 shards): on
CPU it must reproduce the oracle's search exactly for a correct index, and
flag a wrong rank, a wrong window and an unsorted neighbourhood."""
import numpy as np

from oracle import certify as CE
from oracle import pyoracle as P

N = 4000


class _OracleIndex:
    """An 'index' backed by the CPU oracle, with optional corruption."""

    def __init__(self, view, m, bad=None):
        self.rows = P.gen_rows(0, N)
        self.oi = P.Oracle(P.view_floats(self.rows, view), 8, m)
        self.view = view
        self.bad = bad

    def size(self):
        return N

    def curves(self):
        return 8

    def windows(self, qs, depth):
        r, b, e = self.oi.windows(P.view_floats(qs, self.view), depth)
        if self.bad == "rank":
            r = r.copy()
            r[0, 3] = min(int(r[0, 3]) + 5, N)
        if self.bad == "window":
            b = b.copy()
            e = e.copy()
            if b[0, 2] > 0:
                b[0, 2] -= 1
                e[0, 2] -= 1
            else:
                b[0, 2] += 1
                e[0, 2] += 1
        return r, b, e

    def sorted_ids(self, c, begin, count):
        ids = self.oi.sorted(c)[1][begin:begin + count].copy()
        if self.bad == "order" and c == 1 and count > 3:
            ids[1], ids[2] = ids[2], ids[1]
        return ids


def test_certificate_reproduces_the_oracle():
    for view, m in ((P.LIFTED, 16), (P.RAW, 8)):
        ix = _OracleIndex(view, m)
        qs = P.gen_queries(0, 25, N)
        ids, dist, ln, rep = CE.certify_shard(ix, qs, 350, 10, view, m)
        oids, od, ol = ix.oi.search(P.view_floats(qs, view), 10, 350)
        assert sum(rep["failed_checks"].values()) == 0
        np.testing.assert_array_equal(ids, oids)
        assert dist.tobytes() == od.tobytes()
        np.testing.assert_array_equal(ln, ol)


def test_certificate_flags_corruption():
    qs = P.gen_queries(0, 3, N)
    for bad, field in (("rank", "lower_bound"), ("window", "window_rule"), ("order", "sorted_neighbourhood")):
        _, _, _, rep = CE.certify_shard(_OracleIndex(P.LIFTED, 16, bad), qs, 64, 10, P.LIFTED, 16)
        assert rep["failed_checks"][field] > 0, (bad, rep)


def test_shard_merge_matches_sharded_oracle():
    rows = P.gen_rows(0, N)
    qs = P.gen_queries(0, 10, N)
    parts = []
    for r in range(3):
        sel = np.arange(r, N, 3, dtype=np.uint64)
        oi = P.Oracle(P.view_floats(rows[sel.astype(np.int64)], P.LIFTED), 8, 16, ids=sel)
        parts.append(oi.search(P.view_floats(qs, P.LIFTED), 10, 100))
    ids, dist, ln = P.merge_shard_lists(parts, 10)
    oids, od, ol = P.sharded_search(P.view_floats(rows, P.LIFTED), P.view_floats(qs, P.LIFTED), 3, 8, 16, 10, 100)
    np.testing.assert_array_equal(ids, oids)
    assert dist.tobytes() == od.tobytes()
