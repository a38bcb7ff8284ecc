"""Regenerate tests/golden/ref_fixture.npz from the REFERENCE itself.

Runs the unmodified reference TUs (/root/reference/proj/src/curve.cpp and
vecio.cpp, compiled by oracle/Makefile into oracle/_ref/libhcref.so together
with the multicurves.hpp restatement) on small synthetic inputs and stores
their outputs.  tests/test_oracle.py checks the independent restatement
(oracle/liboracle.so) against these vectors, so the oracle stays pinned even
where the reference tree is absent (the GPU box).

    python tests/golden/make_golden.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_fixture.npz")


def main():
    if not P.ref_available():
        P.build_oracle()
    assert P.ref_available(), "oracle/_ref/libhcref.so needs /root/reference"
    n, nq, NC = 2000, 24, 8
    rows = P.gen_rows(0, n, 1)
    qs = P.gen_queries(0, nq, n, 1)
    qs[0] = rows[123]  # a self-query
    out = {"rows": rows, "queries": qs}
    # quantizer over every byte, both views, several m (curve.cpp:166-174)
    for view in (P.RAW, P.LIFTED):
        f = P.view_floats(np.arange(256, dtype=np.uint8), view)
        for m in (8, 12, 16, 17, 20, 24, 32):
            cells = []
            for x in f:
                v = ctypes.c_uint64()
                assert P.ref().ref_quantize(ctypes.c_float(float(x)), m, ctypes.byref(v)) == 0
                cells.append(v.value)
            out[f"quant_v{view}_m{m}"] = np.array(cells, np.uint64)
    # curve keys of random points (curve.cpp:62-164)
    rng = np.random.default_rng(7)
    for kind in (P.ZORDER, P.HILBERT):
        for d, m in ((2, 8), (3, 5), (16, 8), (16, 16), (8, 32), (128, 8), (64, 16)):
            pts = rng.integers(0, 1 << m, size=(40, d), dtype=np.uint64)
            keys = np.zeros((40, 16), np.uint64)
            for i in range(40):
                assert P.ref().ref_curve_encode(kind, d, m, np.ascontiguousarray(pts[i]), keys[i]) == 0
            out[f"pts_k{kind}_d{d}_m{m}"] = pts
            out[f"keys_k{kind}_d{d}_m{m}"] = keys
    # index build / windows / candidates / search / brute force (multicurves.hpp, vecio.cpp)
    for view, m in ((P.RAW, 8), (P.LIFTED, 16)):
        for kind in (P.HILBERT, P.ZORDER):
            tag = f"v{view}_k{kind}"
            ri = P.RefIndex(rows, NC, m, kind, view)
            words = (128 // NC * m + 63) // 64
            for c in (0, 3, 7):
                keys, ids = ri.sorted(c, words)
                out[f"sorted_ids_{tag}_c{c}"] = ids
                out[f"sorted_keys_{tag}_c{c}"] = keys
            for depth in (1, 7, 64, 350, 5000):
                r, b, e = ri.windows(qs, depth)
                out[f"win_{tag}_d{depth}"] = np.stack([r, b, e])
            for depth in (7, 350):
                out[f"cand_{tag}_d{depth}_q5"] = ri.candidates(qs[5], depth)
            for k, depth in ((10, 64), (10, 350), (100, 350), (1, 1)):
                ids, dist, ln = ri.search(qs, k, depth, threads=1)
                out[f"search_{tag}_k{k}_d{depth}"] = ids
                out[f"searchd_{tag}_k{k}_d{depth}"] = dist
                out[f"searchl_{tag}_k{k}_d{depth}"] = ln
            if kind == P.HILBERT:
                ids, dist, ln = ri.brute_force(qs, 10, threads=1)
                out[f"brute_v{view}"] = ids
                out[f"bruted_v{view}"] = dist
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
