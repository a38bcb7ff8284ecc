"""ctypes/numpy front-end to the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module, and only as the checker or as the timed CPU baseline.
The product package (paper_1209_0410_b200) never imports it.

Two back ends with the same argument meaning:
  Oracle    -> oracle/liboracle.so       (independent restatement, hc_oracle.cpp)
  RefIndex  -> oracle/_ref/libhcref.so   (reference curve.cpp/vecio.cpp + the
               multicurves.hpp definitions in ref_multicurves.cpp)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhcref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

RAW, LIFTED = 0, 1
ZORDER, HILBERT = 0, 1


def build_oracle() -> None:
    """Compile liboracle.so (and _ref/libhcref.so when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def view_floats(rows_u8: np.ndarray, view: int) -> np.ndarray:
    """Float components the reference sees for byte rows in a given view.

    raw    : float(b)        (bvecs widening, vecio.cpp:50-51)
    lifted : 1 + b/256       (exact in f32)
    """
    f = rows_u8.astype(np.float32)
    if view == LIFTED:
        f = np.float32(1.0) + f / np.float32(256.0)
    return np.ascontiguousarray(f, dtype=np.float32)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
    return C.CDLL(path)


_orc = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        L = _load(ORACLE_SO)
        L.orc_float_to_ordinal.restype = C.c_uint32
        L.orc_float_to_ordinal.argtypes = [C.c_float]
        L.orc_quantize.argtypes = [C.c_float, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_curve_encode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.orc_curve_decode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.orc_default_scheme.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p]
        L.orc_build.restype = C.c_void_p
        L.orc_build.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p,
                                _f32p, C.c_uint64, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_size.restype = C.c_uint64
        L.orc_size.argtypes = [C.c_void_p]
        L.orc_key_words.restype = C.c_uint32
        L.orc_key_words.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_sorted.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]
        L.orc_query_key.argtypes = [C.c_void_p, _f32p, C.c_uint32, _u64p]
        L.orc_windows.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.c_uint64, _u64p, _u64p, _u64p]
        L.orc_candidates.restype = C.c_uint64
        L.orc_candidates.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.c_void_p]
        L.orc_search.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                 _u64p, _f64p, _u32p, C.c_int]
        L.orc_brute_force.argtypes = [_f32p, C.c_void_p, C.c_uint64, C.c_uint32, _f32p, C.c_uint64,
                                      C.c_uint64, _u64p, _f64p, _u32p, C.c_int]
        L.orc_gen_rows.argtypes = [C.c_uint64, C.c_uint64, _u8p, C.c_int]
        L.orc_gen_rows_strided.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u8p, C.c_int]
        L.orc_gen_queries.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u8p, C.c_int]
        L.orc_gen_rows_ids.argtypes = [_u64p, C.c_uint64, _u8p, C.c_int]
        L.orc_keys_batch.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.c_uint32, _u64p]
        _orc = L
    return _orc


def nthreads() -> int:
    return max(1, os.cpu_count() or 1)


def gen_rows(i0: int, count: int, threads: int | None = None, stride: int = 1) -> np.ndarray:
    out = np.empty((count, 128), np.uint8)
    orc().orc_gen_rows_strided(i0, stride, count, out, threads or nthreads())
    return out


def gen_rows_ids(ids, threads: int | None = None) -> np.ndarray:
    """Generator rows of arbitrary global ids (SURVEY.md §8(d) is counter-based)."""
    idx = np.ascontiguousarray(ids, np.uint64)
    out = np.zeros((idx.shape[0], 128), np.uint8)
    if idx.shape[0]:
        orc().orc_gen_rows_ids(idx, idx.shape[0], out, threads or nthreads())
    return out


def gen_queries(q0: int, count: int, n_db: int, threads: int | None = None) -> np.ndarray:
    out = np.empty((count, 128), np.uint8)
    orc().orc_gen_queries(q0, count, n_db, out, threads or nthreads())
    return out


def quantize(x: float, m: int) -> int:
    v = C.c_uint64()
    rc = orc().orc_quantize(C.c_float(x), m, C.byref(v))
    if rc:
        raise ValueError(f"quantize rc={rc}")
    return v.value


def curve_encode(kind: int, coords, m: int) -> np.ndarray:
    c = np.ascontiguousarray(coords, dtype=np.uint64)
    key = np.zeros(16, np.uint64)
    rc = orc().orc_curve_encode(kind, len(c), m, c, key)
    if rc:
        raise ValueError(f"curve_encode rc={rc}")
    return key


def curve_decode(kind: int, key, d: int, m: int) -> np.ndarray:
    k = np.zeros(16, np.uint64)
    kk = np.asarray(key, dtype=np.uint64)
    k[: len(kk)] = kk
    out = np.zeros(d, np.uint64)
    rc = orc().orc_curve_decode(kind, d, m, k, out)
    if rc:
        raise ValueError(f"curve_decode rc={rc}")
    return out


def key_hex(words) -> str:
    """ExtendedKey::to_hex (curve.cpp:11-27): leading zero words skipped."""
    w = [int(x) for x in words]
    i = len(w) - 1
    while i > 0 and w[i] == 0:
        i -= 1
    s = format(w[i], "x")
    for j in range(i - 1, -1, -1):
        s += format(w[j], "016x")
    return s


def default_scheme(d_full: int, curves: int):
    off = np.zeros(curves + 1, np.uint32)
    asg = np.zeros(d_full, np.uint32)
    if orc().orc_default_scheme(d_full, curves, off, asg):
        raise ValueError("bad scheme")
    return off, asg


class Oracle:
    """The restated MulticurvesIndex over float components (multicurves.hpp:74-107)."""

    def __init__(self, rows_f32: np.ndarray, curves: int, m: int, kind: int = HILBERT,
                 ids: np.ndarray | None = None, off=None, assign=None, threads: int | None = None):
        rows = np.ascontiguousarray(rows_f32, dtype=np.float32)
        self.n, self.d = rows.shape
        if off is None:
            off, assign = default_scheme(self.d, curves)
        self.off = np.ascontiguousarray(off, np.uint32)
        self.assign = np.ascontiguousarray(assign, np.uint32)
        self.curves = len(self.off) - 1
        self._ids = None if ids is None else np.ascontiguousarray(ids, np.uint64)
        err = C.c_int()
        idp = None if self._ids is None else self._ids.ctypes.data
        self.h = orc().orc_build(self.d, self.curves, m, kind, self.off, self.assign, rows,
                                 self.n, idp, threads or nthreads(), C.byref(err))
        if not self.h:
            raise ValueError(f"orc_build rc={err.value}")

    def __del__(self):
        if getattr(self, "h", None):
            orc().orc_free(self.h)
            self.h = None

    def words(self, c: int) -> int:
        return orc().orc_key_words(self.h, c)

    def sorted(self, c: int):
        w = self.words(c)
        keys = np.zeros((self.n, w), np.uint64)
        ids = np.zeros(self.n, np.uint64)
        orc().orc_sorted(self.h, c, keys.ctypes.data, ids.ctypes.data)
        return keys, ids

    def query_key(self, q_f32: np.ndarray, c: int) -> np.ndarray:
        key = np.zeros(16, np.uint64)
        rc = orc().orc_query_key(self.h, np.ascontiguousarray(q_f32, np.float32), c, key)
        if rc:
            raise ValueError(f"query_key rc={rc}")
        return key

    def keys(self, rows_f32: np.ndarray, c: int) -> np.ndarray:
        """Full keys [n, words] (LS word first) of arbitrary rows on curve c."""
        rows = np.ascontiguousarray(rows_f32, np.float32)
        out = np.zeros((rows.shape[0], self.words(c)), np.uint64)
        if rows.shape[0]:
            rc = orc().orc_keys_batch(self.h, rows, rows.shape[0], c, out)
            if rc:
                raise ValueError(f"keys rc={rc}")
        return out

    def windows(self, qs_f32: np.ndarray, depth: int):
        qs = np.ascontiguousarray(qs_f32, np.float32)
        nq = qs.shape[0]
        r = np.zeros(nq * self.curves, np.uint64)
        b = np.zeros_like(r)
        e = np.zeros_like(r)
        rc = orc().orc_windows(self.h, qs, nq, depth, r, b, e)
        if rc:
            raise ValueError(f"windows rc={rc}")
        shp = (nq, self.curves)
        return r.reshape(shp), b.reshape(shp), e.reshape(shp)

    def candidates(self, q_f32: np.ndarray, depth: int) -> np.ndarray:
        q = np.ascontiguousarray(q_f32, np.float32)
        out = np.zeros(self.curves * min(depth, self.n) + 1, np.uint64)
        n = orc().orc_candidates(self.h, q, depth, out.ctypes.data)
        return out[:n]

    def search(self, qs_f32: np.ndarray, k: int, depth: int, threads: int | None = None):
        qs = np.ascontiguousarray(qs_f32, np.float32)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        dist = np.zeros((nq, k), np.float64)
        ln = np.zeros(nq, np.uint32)
        rc = orc().orc_search(self.h, qs, nq, k, depth, ids, dist, ln, threads or nthreads())
        if rc:
            raise ValueError(f"search rc={rc}")
        return ids, dist, ln


def brute_force(rows_f32: np.ndarray, qs_f32: np.ndarray, k: int, ids=None, threads: int | None = None):
    rows = np.ascontiguousarray(rows_f32, np.float32)
    qs = np.ascontiguousarray(qs_f32, np.float32)
    nq = qs.shape[0]
    oi = np.zeros((nq, k), np.uint64)
    od = np.zeros((nq, k), np.float64)
    ln = np.zeros(nq, np.uint32)
    idv = None if ids is None else np.ascontiguousarray(ids, np.uint64)
    rc = orc().orc_brute_force(rows, None if idv is None else idv.ctypes.data, rows.shape[0],
                               rows.shape[1], qs, nq, k, oi, od, ln, threads or nthreads())
    if rc:
        raise ValueError(f"brute_force rc={rc}")
    return oi, od, ln


def sharded_search(rows_f32: np.ndarray, qs_f32: np.ndarray, shards: int, curves: int, m: int,
                   k: int, depth: int, kind: int = HILBERT):
    """Sharded oracle: partition by id mod G,
    per-shard search at the per-shard depth, then a (distance, id) merge
    truncated to k."""
    n = rows_f32.shape[0]
    gid = np.arange(n, dtype=np.uint64)
    parts = []
    for s in range(shards):
        sel = gid % shards == s
        if not sel.any():
            continue
        ix = Oracle(rows_f32[sel], curves, m, kind, ids=gid[sel])
        parts.append(ix.search(qs_f32, k, depth))
    nq = qs_f32.shape[0]
    oi = np.zeros((nq, k), np.uint64)
    od = np.zeros((nq, k), np.float64)
    ln = np.zeros(nq, np.uint32)
    for q in range(nq):
        pool = []
        for ids, dist, l in parts:
            pool += [(dist[q, i], int(ids[q, i])) for i in range(l[q])]
        pool.sort()
        pool = pool[:k]
        ln[q] = len(pool)
        for i, (d, j) in enumerate(pool):
            oi[q, i] = j
            od[q, i] = d
    return oi, od, ln


# ---------------------------------------------------------------------------
# Reference TUs (oracle/_ref) -- only where the reference tree was present at
# build time; the built .so travels with the snapshot.
# ---------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = _load(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_float_to_ordinal.restype = C.c_uint32
        L.ref_float_to_ordinal.argtypes = [C.c_float, C.POINTER(C.c_int)]
        L.ref_quantize.argtypes = [C.c_float, C.c_uint32, C.POINTER(C.c_uint64)]
        L.ref_curve_encode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.ref_curve_decode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.ref_build.restype = C.c_void_p
        L.ref_build.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u8p, C.c_uint64,
                                C.c_int, C.POINTER(C.c_int)]
        L.ref_build_ids.restype = C.c_void_p
        L.ref_build_ids.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u8p, C.c_uint64,
                                    C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_sorted.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
        L.ref_windows.argtypes = [C.c_void_p, _u8p, C.c_uint64, C.c_uint64, _u64p, _u64p, _u64p]
        L.ref_candidates.restype = C.c_uint64
        L.ref_candidates.argtypes = [C.c_void_p, _u8p, C.c_uint64, C.c_void_p]
        L.ref_search.argtypes = [C.c_void_p, _u8p, C.c_uint64, C.c_uint64, C.c_uint64, _u64p,
                                 _f64p, _u32p, C.c_int]
        L.ref_brute_force.argtypes = [C.c_void_p, _u8p, C.c_uint64, C.c_uint64, _u64p, _f64p,
                                      _u32p, C.c_int]
        L.ref_select_top_k.argtypes = [_u64p, _f64p, C.c_uint64, C.c_uint64, _u64p, _f64p]
        _ref = L
    return _ref


def ref_error() -> str:
    return ref().ref_last_error().decode()


class RefIndex:
    """hc::MulticurvesIndex from the reference TUs, over byte rows in a view."""

    def __init__(self, rows_u8: np.ndarray, curves: int, m: int, kind: int = HILBERT, view: int = RAW,
                 id_base: int = 0, id_stride: int = 1):
        """id_base / id_stride: row i has id id_base + i * id_stride (one shard
        of the id mod G partition)."""
        rows = np.ascontiguousarray(rows_u8, np.uint8)
        self.n, self.d = rows.shape
        self.curves = curves
        self.view = view
        err = C.c_int()
        if id_base == 0 and id_stride == 1:
            self.h = ref().ref_build(self.d, curves, m, kind, rows, self.n, view, C.byref(err))
        else:
            self.h = ref().ref_build_ids(self.d, curves, m, kind, rows, self.n, view, id_base, id_stride,
                                         C.byref(err))
        if not self.h:
            raise ValueError(f"ref_build: {ref_error()}")

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_free(self.h)
            self.h = None

    def sorted(self, c: int, words: int):
        keys = np.zeros((self.n, words), np.uint64)
        ids = np.zeros(self.n, np.uint64)
        ref().ref_sorted(self.h, c, words, keys.ctypes.data, ids.ctypes.data)
        return keys, ids

    def windows(self, qs_u8: np.ndarray, depth: int):
        qs = np.ascontiguousarray(qs_u8, np.uint8)
        nq = qs.shape[0]
        r = np.zeros(nq * self.curves, np.uint64)
        b = np.zeros_like(r)
        e = np.zeros_like(r)
        if ref().ref_windows(self.h, qs, nq, depth, r, b, e):
            raise ValueError(ref_error())
        shp = (nq, self.curves)
        return r.reshape(shp), b.reshape(shp), e.reshape(shp)

    def candidates(self, q_u8: np.ndarray, depth: int) -> np.ndarray:
        out = np.zeros(self.curves * min(depth, self.n) + 1, np.uint64)
        n = ref().ref_candidates(self.h, np.ascontiguousarray(q_u8, np.uint8), depth, out.ctypes.data)
        return out[:n]

    def search(self, qs_u8: np.ndarray, k: int, depth: int, threads: int | None = None):
        qs = np.ascontiguousarray(qs_u8, np.uint8)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        dist = np.zeros((nq, k), np.float64)
        ln = np.zeros(nq, np.uint32)
        if ref().ref_search(self.h, qs, nq, k, depth, ids, dist, ln, threads or nthreads()):
            raise ValueError(ref_error())
        return ids, dist, ln

    def brute_force(self, qs_u8: np.ndarray, k: int, threads: int | None = None):
        qs = np.ascontiguousarray(qs_u8, np.uint8)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        dist = np.zeros((nq, k), np.float64)
        ln = np.zeros(nq, np.uint32)
        if ref().ref_brute_force(self.h, qs, nq, k, ids, dist, ln, threads or nthreads()):
            raise ValueError(ref_error())
        return ids, dist, ln


def merge_shard_lists(parts, k: int):
    """Hypershard aggregate over per-shard (ids, dist, len) results: (distance,
    id) order, truncated to k, vectorised over queries."""
    nq = parts[0][0].shape[0]
    ids = np.concatenate([p[0][:, :k] for p in parts], axis=1)
    dist = np.concatenate([p[1][:, :k] for p in parts], axis=1)
    valid = np.concatenate([np.arange(k)[None, :] < p[2][:, None] for p in parts], axis=1)
    dist = np.where(valid, dist, np.inf)
    ids = np.where(valid, ids, np.uint64(2**64 - 1))
    oi = np.zeros((nq, k), np.uint64)
    od = np.zeros((nq, k), np.float64)
    ln = np.minimum(valid.sum(axis=1), k).astype(np.uint32)
    for q in range(nq):
        order = np.lexsort((ids[q], dist[q]))[:k]
        oi[q] = ids[q, order]
        od[q] = dist[q, order]
    return oi, od, ln


def ref_sharded_search(n_total: int, shards: int, qs_u8: np.ndarray, curves: int, m: int, kind: int, view: int,
                       k: int, depths, threads: int | None = None):
    """The reference's sharded search on the generator's rows: shard r holds
    global ids r, r + G, ..., each shard is an
    hc::MulticurvesIndex built from the reference TUs and searched at the
    per-shard depth, and the per-shard lists are merged by (distance, id).
    One shard is resident at a time.  depths: int or list; returns the merged
    (ids, dist, len) per depth (a dict for a list)."""
    ds = [depths] if isinstance(depths, int) else list(depths)
    parts = {d: [] for d in ds}
    for r in range(shards):
        cnt = 0 if r >= n_total else (n_total - r + shards - 1) // shards
        rows = gen_rows(r, cnt, threads, stride=shards)
        ri = RefIndex(rows, curves, m, kind, view, id_base=r, id_stride=shards)
        del rows
        for d in ds:
            parts[d].append(ri.search(qs_u8, k, d, threads))
        del ri
    out = {d: merge_shard_lists(parts[d], k) for d in ds}
    return out[ds[0]] if isinstance(depths, int) else out
