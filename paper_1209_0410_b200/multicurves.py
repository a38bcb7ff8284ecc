"""Host-side mirror of the reference's index interface over the C ABI.

Names and argument meaning follow the reference's namespace hc
(proj/include/hypercurves/multicurves.hpp, vecio.hpp, curve.hpp):
ProjectionScheme, default_scheme, SearchParams, Neighbor, MulticurvesIndex
with search / retrieve_candidates / candidate_union / subindex taps, and
brute_force_knn.  Errors the reference raises as std::invalid_argument come
back as HcgInvalidArgument (a ValueError).

Buffers may be numpy arrays (host) or torch tensors (host or CUDA); outputs
follow the queries: CUDA tensors in -> CUDA tensors out, else numpy.
Everything runs on the sm_100a kernels in libhcg.so -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from ._lib import HCG_F32, HCG_HILBERT, HCG_U8, HCG_ZORDER, HcgInvalidArgument, HcgScheme, check, lib

ZORDER, HILBERT = HCG_ZORDER, HCG_HILBERT


@dataclass(frozen=True)
class View:
    """How the reference sees a descriptor byte b: offset + b * scale (f32).

    raw    : float(b)          -- bvecs widening (vecio.cpp:50-51)
    lifted : 1 + b/256         -- SURVEY.md F4; the reference quantizer keeps
                                  the byte order at m >= 16
    """
    offset: float
    scale: float
    name: str

    def floats(self, rows_u8: np.ndarray) -> np.ndarray:
        f = np.asarray(rows_u8).astype(np.float32)
        if self.scale != 1.0:
            f = f * np.float32(self.scale)
        if self.offset != 0.0:
            f = np.float32(self.offset) + f
        return f


RAW = View(0.0, 1.0, "raw")
LIFTED = View(1.0, 1.0 / 256.0, "lifted")


@dataclass
class ProjectionScheme:
    """multicurves.hpp:18-32."""
    d_full: int
    bits_per_dim: int = 8
    curve_kind: int = HILBERT
    seed: int = 0
    assignment: list = field(default_factory=list)

    def curves(self) -> int:
        return len(self.assignment)

    def dims_of(self, c: int) -> int:
        return len(self.assignment[c])


def default_scheme(d_full: int, curves: int, bits_per_dim: int = 8, kind: int = HILBERT,
                   seed: int = 0) -> ProjectionScheme:
    """Round-robin dims over curves.  The seeded permutation
    (seed != 0) is unpinned by the reference and rejected."""
    if seed != 0:
        raise HcgInvalidArgument(-1, "seeded permutation is unpinned by the reference (SPEC.md:203)")
    off = (C.c_uint32 * (curves + 1))()
    asg = (C.c_uint32 * max(d_full, 1))()
    check(lib().hcg_default_assignment(d_full, curves, off, asg))
    assignment = [[int(asg[i]) for i in range(off[c], off[c + 1])] for c in range(curves)]
    return ProjectionScheme(d_full, bits_per_dim, kind, seed, assignment)


@dataclass
class SearchParams:
    """multicurves.hpp:69-72."""
    k: int = 1
    probe_depth: int = 1


class Neighbor(NamedTuple):
    """vecio.hpp:27-32: id and rooted Euclidean distance."""
    id: int
    distance: float


def make_lut(view: View, bits_per_dim: int) -> np.ndarray:
    lut = (C.c_uint32 * 256)()
    check(lib().hcg_make_lut(C.c_float(view.offset), C.c_float(view.scale), bits_per_dim, lut))
    return np.frombuffer(lut, dtype=np.uint32).copy()


def c_scheme(scheme: "ProjectionScheme", view: View, dtype: str = "u8") -> HcgScheme:
    """The hcg_scheme of a ProjectionScheme seen through `view` (the assignment
    arrays stay alive with the returned struct)."""
    off = [0]
    flat = []
    for slots in scheme.assignment:
        flat += list(slots)
        off.append(len(flat))
    s = HcgScheme()
    s._off = (C.c_uint32 * len(off))(*off)
    s._asg = (C.c_uint32 * max(len(flat), 1))(*flat)
    s.d_full = scheme.d_full
    s.curves = scheme.curves()
    s.bits_per_dim = scheme.bits_per_dim
    s.curve_kind = scheme.curve_kind
    s.assign_off = s._off
    s.assign = s._asg
    lut = make_lut(view, scheme.bits_per_dim)
    for b in range(256):
        s.cell_lut[b] = int(lut[b])
    s.dist_scale = float(view.scale) if dtype == "u8" else 1.0
    s.dtype = HCG_U8 if dtype == "u8" else HCG_F32
    s.view_offset = float(view.offset) if dtype == "u8" else 0.0
    return s


# ----------------------------------------------------------------- buffers ----
def _torch():
    import torch
    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _is_cuda(x) -> bool:
    return _is_torch(x) and x.is_cuda


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise HcgInvalidArgument(-1, "tensor must be contiguous")
        return x.data_ptr()
    if not x.flags["C_CONTIGUOUS"]:
        raise HcgInvalidArgument(-1, "array must be C-contiguous")
    return x.ctypes.data


def _u8_2d(x, d_full: int, dtype: str = "u8"):
    """Validate n x d_full descriptors of the index's element type (u8 / f32)."""
    np_dt = np.uint8 if dtype == "u8" else np.float32
    if _is_torch(x):
        torch = _torch()
        if x.dtype != (torch.uint8 if dtype == "u8" else torch.float32):
            raise HcgInvalidArgument(-1, f"descriptors must be {np.dtype(np_dt).name}")
        x = x.contiguous()
        if x.dim() == 1:
            x = x.view(1, -1)
    else:
        x = np.ascontiguousarray(x)
        if x.dtype != np_dt:
            raise HcgInvalidArgument(-1, f"descriptors must be {np.dtype(np_dt).name}")
        if x.ndim == 1:
            x = x.reshape(1, -1)
    if x.shape[1] != d_full:
        raise HcgInvalidArgument(-1, f"dimension mismatch: {x.shape[1]} vs {d_full}")
    return x


def _empty_like_kind(ref, shape, np_dtype):
    if _is_cuda(ref):
        torch = _torch()
        tdt = {np.uint64: torch.uint64, np.uint32: torch.uint32, np.int64: torch.int64,
               np.float64: torch.float64}[np_dtype]
        return torch.empty(shape, dtype=tdt, device=ref.device)
    return np.empty(shape, dtype=np_dtype)


def _stream(stream, ref=None):
    if stream is not None:
        return stream if isinstance(stream, int) else int(stream.cuda_stream)
    if ref is not None and _is_cuda(ref):
        return int(_torch().cuda.current_stream(ref.device).cuda_stream)
    return None


# ------------------------------------------------------------------- index ----
class MulticurvesIndex:
    """hc::MulticurvesIndex (multicurves.hpp:74-107) resident on one B200.

    rows: n x d_full descriptors (numpy or torch, host or device) -- uint8
    (bvecs, seen through `view`) or float32 (the reference's own component
    type, fvecs; `view` unused); the id of row s is id_base + s * id_stride
    (ids 0..n-1 by default).  dtype ("u8" / "f32") defaults to the rows'.
    """

    def __init__(self, rows, scheme: ProjectionScheme, view: View = RAW, device: int = 0,
                 id_base: int = 0, id_stride: int = 1, stream=None, _handle=None, dtype: str | None = None):
        self.scheme = scheme
        self.view = view
        self.device = device
        self.id_base = id_base
        self.id_stride = id_stride
        self._h = None
        if _handle is not None:  # MulticurvesIndex.load
            self._h = _handle
            self.dtype = "f32" if lib().hcg_index_dtype(_handle) == HCG_F32 else "u8"
            return
        if dtype is None:
            is_f32 = rows is not None and str(getattr(rows, "dtype", "")).endswith("float32")
            dtype = "f32" if is_f32 else "u8"
        if dtype not in ("u8", "f32"):
            raise HcgInvalidArgument(-1, f"unknown descriptor dtype {dtype!r}")
        self.dtype = dtype
        d = scheme.d_full
        rows = (_u8_2d(rows, d, dtype) if (rows is not None and len(rows))
                else np.zeros((0, d), np.uint8 if dtype == "u8" else np.float32))
        n = rows.shape[0]
        s = c_scheme(scheme, view, dtype)
        self._scheme_c = s
        h = C.c_void_p()
        check(lib().hcg_build(C.byref(s), _ptr(rows), n, id_base, id_stride, device,
                              _stream(stream, rows), C.byref(h)))
        self._h = h

    def _rows(self, x):
        return _u8_2d(x, self.scheme.d_full, self.dtype)

    # -- growth and persistence
    def insert(self, rows, stream=None) -> None:
        """multicurves.hpp:79, batched: append rows (ids continue id_base + s*id_stride)."""
        r = self._rows(rows)
        check(lib().hcg_insert(self._h, _ptr(r), r.shape[0], _stream(stream, r)))

    def save(self, path: str) -> None:
        """multicurves.hpp:96-97: little-endian, bit-exact round trip."""
        check(lib().hcg_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, scheme: ProjectionScheme | None = None, view: View | None = None, device: int = 0,
             id_base: int = 0, id_stride: int = 1) -> "MulticurvesIndex":
        """multicurves.hpp:98.  The file carries the scheme and the view; when
        `scheme` / `view` are omitted they are read back from the index."""
        h = C.c_void_p()
        check(lib().hcg_load(os.fsencode(path), device, None, C.byref(h)))
        if scheme is None or view is None:
            s = HcgScheme()
            n_asg = C.c_uint32()
            check(lib().hcg_describe(h, C.byref(s), None, None, C.byref(n_asg)))
            off = (C.c_uint32 * (s.curves + 1))()
            asg = (C.c_uint32 * max(n_asg.value, 1))()
            check(lib().hcg_describe(h, C.byref(s), off, asg, C.byref(n_asg)))
            if scheme is None:
                scheme = ProjectionScheme(s.d_full, s.bits_per_dim, s.curve_kind, 0,
                                          [[int(asg[i]) for i in range(off[c], off[c + 1])] for c in range(s.curves)])
            if view is None:
                view = View(float(s.view_offset), float(s.dist_scale), "loaded")
        return cls(None, scheme, view, device, id_base, id_stride, _handle=h)

    # -- lifetime
    def close(self) -> None:
        if self._h:
            lib().hcg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- shape
    def size(self) -> int:
        return int(lib().hcg_size(self._h))

    def curves(self) -> int:
        return int(lib().hcg_curves(self._h))

    def key_words(self, c: int) -> int:
        return int(lib().hcg_key_words(self._h, c))

    def unionless(self, nq: int, k: int, depth: int) -> bool:
        """Whether a search of nq queries runs the union-less refine kernel."""
        return bool(lib().hcg_refine_unionless(self._h, nq, k, depth))

    def device_bytes(self) -> int:
        return int(lib().hcg_device_bytes(self._h))

    def rooted(self, sqdist) -> np.ndarray:
        """Reference distance (vecio.cpp:111): sqrt of the exact squared distance."""
        s = np.asarray(sqdist.cpu() if _is_torch(sqdist) else sqdist).astype(np.float64)
        return np.sqrt(s) * (self.view.scale if self.dtype == "u8" else 1.0)

    # -- batched search (the hot path)
    def search_batch(self, queries, k: int, probe_depth: int, stream=None, out=None):
        """Top-k by (distance, id) of every query: (ids u64 [nq,k], sqdist
        [nq,k], len u32 [nq]).  sqdist is u32 (exact integers) for u8 rows,
        padded with 2^32-1; f64 for f32 rows, padded with +inf.  Padding ids
        are 2^64-1."""
        q = self._rows(queries)
        nq = q.shape[0]
        f32 = self.dtype == "f32"
        if out is None:
            ids = _empty_like_kind(q, (nq, k), np.uint64)
            sq = _empty_like_kind(q, (nq, k), np.float64 if f32 else np.uint32)
            ln = _empty_like_kind(q, (nq,), np.uint32)
        else:
            ids, sq, ln = out
        fn = lib().hcg_search_f32 if f32 else lib().hcg_search
        check(fn(self._h, _ptr(q), nq, k, probe_depth, _ptr(ids), _ptr(sq), _ptr(ln), _stream(stream, q)))
        return ids, sq, ln

    def search_timed(self, queries, k: int, probe_depth: int, out, stream=None):
        """search_batch into preallocated outputs, returning the device times (ms)
        of (locate, candidate union, gather+score) measured with CUDA events on `stream`."""
        q = self._rows(queries)
        ids, sq, ln = out
        ms = (C.c_float * 3)()
        check(lib().hcg_search_timed(self._h, _ptr(q), q.shape[0], k, probe_depth, _ptr(ids), _ptr(sq),
                                     _ptr(ln), ms, _stream(stream, q)))
        return float(ms[0]), float(ms[1]), float(ms[2])

    def search(self, query, params: SearchParams) -> list:
        """hc::MulticurvesIndex::search for one query -> NeighborList."""
        ids, sq, ln = self.search_batch(query, params.k, params.probe_depth)
        ids = np.asarray(ids.cpu() if _is_torch(ids) else ids)[0]
        d = self.rooted(sq)[0]
        n = int(np.asarray(ln.cpu() if _is_torch(ln) else ln)[0])
        return [Neighbor(int(ids[i]), float(d[i])) for i in range(n)]

    def search_packed(self, queries, k: int, probe_depth: int, out=None, stream=None):
        """Per-shard packed results (sqdist<<32 | id) for the sharded merge."""
        q = self._rows(queries)
        nq = q.shape[0]
        if out is None:
            out = _empty_like_kind(q, (nq, k), np.uint64)
        check(lib().hcg_search_packed(self._h, _ptr(q), nq, k, probe_depth, _ptr(out),
                                      _stream(stream, q)))
        return out

    # -- parity taps
    def keys(self, rows, c: int) -> np.ndarray:
        """curve_encode(kind, project(v, scheme, c)) of each row: [n, words] u64 (LS word first)."""
        r = self._rows(rows)
        out = np.zeros((r.shape[0], self.key_words(c)), np.uint64)
        check(lib().hcg_keys(self._h, _ptr(r), r.shape[0], c, _ptr(out), _stream(None, r)))
        return out

    def subindex(self, c: int, with_keys: bool = False):
        """SubIndex::entries() of curve c: ids (and full keys) in sorted order."""
        n = self.size()
        ids = np.zeros(n, np.uint64)
        keys = np.zeros((n, self.key_words(c)), np.uint64) if with_keys else None
        check(lib().hcg_sorted(self._h, c, _ptr(ids), _ptr(keys) if with_keys else None, None))
        return (ids, keys) if with_keys else ids

    def windows(self, queries, probe_depth: int):
        """rank_of and window [begin, end) per (query, curve)."""
        q = self._rows(queries)
        nq, C_ = q.shape[0], self.curves()
        r = np.zeros((nq, C_), np.uint64)
        b = np.zeros((nq, C_), np.uint64)
        e = np.zeros((nq, C_), np.uint64)
        check(lib().hcg_windows(self._h, _ptr(q), nq, probe_depth, _ptr(r), _ptr(b), _ptr(e),
                                _stream(None, q)))
        return r, b, e

    def sorted_ids(self, c: int, begin: int, count: int) -> np.ndarray:
        """Ids at positions [begin, begin + count) of sorted subindex c (SubIndex::entries() slice)."""
        out = np.zeros(max(count, 1), np.uint64)
        if count:
            check(lib().hcg_sorted_range(self._h, c, begin, count, _ptr(out), None))
        return out[:count]

    def retrieve_candidates(self, query, c: int, depth: int) -> np.ndarray:
        """Ids of the window on curve c (multicurves.hpp:83-85), in key order."""
        _, b, e = self.windows(query, depth)
        begin, end = int(b[0, c]), int(e[0, c])
        out = np.zeros(max(end - begin, 1), np.uint64)
        check(lib().hcg_sorted_range(self._h, c, begin, end - begin, _ptr(out), None))
        return out[:end - begin]

    def candidates(self, queries, probe_depth: int):
        """Deduplicated candidate ids per query (list of sorted arrays)."""
        q = self._rows(queries)
        nq = q.shape[0]
        cap = self.curves() * min(probe_depth, max(self.size(), 1))
        out = np.zeros((nq, max(cap, 1)), np.uint64)
        cnt = np.zeros(nq, np.uint32)
        check(lib().hcg_candidates(self._h, _ptr(q), nq, probe_depth, _ptr(out), max(cap, 1),
                                   _ptr(cnt), _stream(None, q)))
        return [np.sort(out[i, :cnt[i]]) for i in range(nq)]

    def candidate_counts(self, queries, probe_depth: int) -> np.ndarray:
        """|candidate_union| per query (unique candidates U_q)."""
        q = self._rows(queries)
        cnt = np.zeros(q.shape[0], np.uint32)
        check(lib().hcg_candidates(self._h, _ptr(q), q.shape[0], probe_depth, None, 0, _ptr(cnt),
                                   _stream(None, q)))
        return cnt

    def candidate_union(self, query, depth: int) -> np.ndarray:
        """multicurves.hpp:87-89 (sorted ascending)."""
        return self.candidates(query, depth)[0]

    def brute_force(self, queries, k: int, stream=None):
        """brute_force_knn (vecio.cpp:115-122) over the indexed rows, on the GPU."""
        q = self._rows(queries)
        nq = q.shape[0]
        f32 = self.dtype == "f32"
        ids = _empty_like_kind(q, (nq, k), np.uint64)
        sq = _empty_like_kind(q, (nq, k), np.float64 if f32 else np.uint32)
        ln = _empty_like_kind(q, (nq,), np.uint32)
        fn = lib().hcg_brute_force_f32 if f32 else lib().hcg_brute_force
        check(fn(self._h, _ptr(q), nq, k, _ptr(ids), _ptr(sq), _ptr(ln), _stream(stream, q)))
        return ids, sq, ln


def read_vectors(path: str, fmt: str = "bvecs", view: View = RAW, dtype: str = "u8") -> np.ndarray:
    """vecio.cpp:18-61: bvecs / fvecs records -> [n, dim] rows: uint8 (the
    view's bytes), or with fmt="fvecs", dtype="f32" the float32 components
    as stored (rows of an f32 index)."""
    from ._lib import HCG_BVECS, HCG_FVECS, HCG_FVECS_F32
    f32 = dtype == "f32"
    if f32 and fmt != "fvecs":
        raise HcgInvalidArgument(-1, "float rows come from fvecs files")
    code = HCG_FVECS_F32 if f32 else (HCG_BVECS if fmt == "bvecs" else HCG_FVECS)
    buf = C.POINTER(C.c_uint8)()
    n = C.c_uint64()
    dim = C.c_uint32()
    check(lib().hcg_read_vectors(os.fsencode(path), code, C.c_float(view.offset), C.c_float(view.scale),
                                 C.byref(buf), C.byref(n), C.byref(dim)))
    try:
        nbytes = n.value * dim.value * (4 if f32 else 1)
        out = np.ctypeslib.as_array(buf, shape=(max(nbytes, 1),))[:nbytes].copy()
    finally:
        lib().hcg_free_buffer(buf)
    dt = np.float32 if f32 else np.uint8
    return out.view(dt).reshape(n.value, dim.value) if n.value else np.zeros((0, dim.value), dt)


def write_vectors(path: str, rows, fmt: str = "bvecs", view: View = RAW) -> None:
    """vecio.cpp:63-85.  float32 rows are written to fvecs as-is."""
    from ._lib import HCG_BVECS, HCG_FVECS, HCG_FVECS_F32
    f32 = np.asarray(rows).dtype == np.float32
    if f32 and fmt != "fvecs":
        raise HcgInvalidArgument(-1, "float rows go to fvecs files")
    r = np.ascontiguousarray(rows, dtype=np.float32 if f32 else np.uint8)
    if r.ndim == 1:
        r = r.reshape(1, -1)
    code = HCG_FVECS_F32 if f32 else (HCG_BVECS if fmt == "bvecs" else HCG_FVECS)
    check(lib().hcg_write_vectors(os.fsencode(path), code, C.c_float(view.offset), C.c_float(view.scale),
                                  _ptr(r), r.shape[0], r.shape[1] if r.size else 0))


def merge_packed(packed, k: int, device: int = 0, stream=None, out=None):
    """Hypershard aggregate: packed [parts, nq, k] -> top-k."""
    parts, nq = int(packed.shape[0]), int(packed.shape[1])
    if out is None:
        ids = _empty_like_kind(packed, (nq, k), np.uint64)
        sq = _empty_like_kind(packed, (nq, k), np.uint32)
        ln = _empty_like_kind(packed, (nq,), np.uint32)
    else:
        ids, sq, ln = out
    check(lib().hcg_merge_packed(_ptr(packed), parts, nq, k, _ptr(ids), _ptr(sq), _ptr(ln), device,
                                 _stream(stream, packed)))
    return ids, sq, ln


# ------------------------------------------------------------ equivalence ----
def binomial_tail(trials: int, p: float, phi: int) -> float:
    if not (0.0 < p < 1.0):
        raise HcgInvalidArgument(-1, "p must be in (0, 1)")
    return float(lib().hcg_binomial_tail(trials, p, phi))


def miss_bound(Phi: int, shards: int, phi: int) -> float:
    return float(lib().hcg_miss_bound(Phi, shards, phi))


def plan_depth(Phi: int, shards: int, target: float) -> int:
    return int(lib().hcg_plan_depth(Phi, shards, target))


def monte_carlo_miss(Phi: int, shards: int, phi: int, trials: int, seed: int = 0) -> float:
    """fraction of trials in which two independent
    Multinomial(Phi, uniform over `shards`) allocations (the two halves of the
    sequential window) put more than phi entries into some shard.  Validates
    miss_bound empirically (§4.2 proof model)."""
    if trials < 1:
        raise HcgInvalidArgument(-1, "trials must be >= 1")
    rng = np.random.default_rng(seed)
    p = np.full(shards, 1.0 / shards)
    misses = 0
    left = trials
    while left:
        b = min(left, 1 << 18)
        lo = rng.multinomial(Phi, p, size=b)
        hi = rng.multinomial(Phi, p, size=b)
        misses += int(((lo > phi).any(axis=1) | (hi > phi).any(axis=1)).sum())
        left -= b
    return misses / trials


def shard_probe_depth(depth: int, shards: int, target: float = 0.02) -> int:
    """Per-shard probe depth 2*phi* for a sequential depth D (Phi = ceil(D/2),
    SPEC.md:329) at a miss-probability target."""
    Phi = (depth + 1) // 2
    return 2 * plan_depth(Phi, shards, target)


# ------------------------------------------------------------- synthetic ----
def gen_rows(first: int, count: int, stride: int = 1, device: int = 0, stream=None):
    """Rows first + i*stride of the SURVEY.md §8(d) generator, as a CUDA uint8 tensor."""
    torch = _torch()
    out = torch.empty((count, 128), dtype=torch.uint8, device=f"cuda:{device}")
    check(lib().hcg_gen_rows(first, stride, count, _ptr(out) if count else None, device,
                             _stream(stream, out)))
    return out


def gen_queries(first: int, count: int, n_db: int, device: int = 0, stream=None):
    torch = _torch()
    out = torch.empty((count, 128), dtype=torch.uint8, device=f"cuda:{device}")
    check(lib().hcg_gen_queries(first, count, n_db, _ptr(out) if count else None, device,
                                _stream(stream, out)))
    return out


def recall_at(found_ids, true_ids, k: int) -> float:
    """Mean |found[:k] ∩ true[:k]| / k over queries."""
    f = np.asarray(found_ids)[:, :k]
    t = np.asarray(true_ids)[:, :k]
    hits = 0
    for a, b in zip(f, t):
        hits += len(set(a.tolist()) & set(b.tolist()) - {2**64 - 1})
    return hits / (k * max(len(f), 1))


def write_search_csv(path: str, ids, distances, lens, query_ids=None) -> int:
    """cmd_search's result file: one `query_id,rank,neighbor_id,distance`
    row per neighbour, rank 0-based within the query's (distance, id)-ordered
    list, distance the rooted double printed with 17 significant digits (round
    trips exactly).  The reference pins the columns, not rank base or number
    format.  Returns the number of rows written."""
    ids = np.asarray(ids.cpu() if _is_torch(ids) else ids)
    dist = np.asarray(distances.cpu() if _is_torch(distances) else distances, dtype=np.float64)
    lens = np.asarray(lens.cpu() if _is_torch(lens) else lens)
    qids = np.arange(len(lens)) if query_ids is None else np.asarray(query_ids)
    rows = 0
    with open(path, "w") as f:
        f.write("query_id,rank,neighbor_id,distance\n")
        for q in range(len(lens)):
            for r in range(int(lens[q])):
                f.write(f"{int(qids[q])},{r},{int(ids[q, r])},{float(dist[q, r]):.17g}\n")
                rows += 1
    return rows


def read_search_csv(path: str):
    """Parse write_search_csv output: list of (query_id, rank, neighbor_id, distance)."""
    out = []
    with open(path) as f:
        header = f.readline().strip()
        if header != "query_id,rank,neighbor_id,distance":
            raise HcgInvalidArgument(-1, f"{path}: not a search CSV")
        for line in f:
            a, b, c, d = line.strip().split(",")
            out.append((int(a), int(b), int(c), float(d)))
    return out


__all__ = [
    "View", "RAW", "LIFTED", "ProjectionScheme", "default_scheme", "SearchParams", "Neighbor",
    "MulticurvesIndex", "merge_packed", "binomial_tail", "miss_bound", "plan_depth",
    "write_search_csv", "read_search_csv", "monte_carlo_miss",
    "shard_probe_depth", "gen_rows", "gen_queries", "make_lut", "recall_at", "ZORDER", "HILBERT",
    "read_vectors", "write_vectors", "c_scheme",
]
