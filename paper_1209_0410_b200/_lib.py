"""ctypes binding of the C ABI in include/hcg.h (libhcg.so, built in-tree).

No fallback: if the CUDA library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HCG_LIB_OVERRIDE: load a differently-compiled libhcg.so (tuning experiments).
LIB_PATH = os.environ.get("HCG_LIB_OVERRIDE") or os.path.join(HERE, "libhcg.so")

HCG_OK = 0
HCG_EINVAL = -1
HCG_ECAPACITY = -2
HCG_ENONFINITE = -3
HCG_ENOMEM = -4
HCG_ECUDA = -5
HCG_ENODEV = -6
HCG_EIO = -7
HCG_FVECS = 0
HCG_BVECS = 1
HCG_FVECS_F32 = 2

HCG_ZORDER = 0
HCG_HILBERT = 1
HCG_MAX_K = 256
HCG_MAX_KEY_BITS = 1024
HCG_U8 = 0
HCG_F32 = 1

# Every symbol include/hcg.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "hcg_last_error", "hcg_version", "hcg_make_lut", "hcg_default_assignment", "hcg_build",
    "hcg_free", "hcg_size", "hcg_curves", "hcg_key_words", "hcg_device_bytes", "hcg_search",
    "hcg_search_timed", "hcg_search_packed", "hcg_merge_packed", "hcg_keys", "hcg_sorted", "hcg_windows",
    "hcg_candidates", "hcg_brute_force", "hcg_binomial_tail", "hcg_miss_bound",
    "hcg_search_f32", "hcg_brute_force_f32", "hcg_index_dtype", "hcg_launch_count", "hcg_sorted_range", "hcg_describe", "hcg_plan_depth", "hcg_gen_rows", "hcg_gen_queries", "hcg_insert", "hcg_save", "hcg_load",
    "hcg_read_vectors", "hcg_write_vectors", "hcg_free_buffer",
    "hcg_nccl_unique_id", "hcg_shard_group_build", "hcg_shard_group_adopt", "hcg_shard_group_join",
    "hcg_shard_group_free", "hcg_shard_group_shards", "hcg_shard_group_search", "hcg_index_device", "hcg_index_ids",
    "hcg_shard_group_device", "hcg_shard_group_dims", "hcg_server_create", "hcg_server_free", "hcg_server_replay",
    "hcg_server_start", "hcg_server_submit", "hcg_server_wait", "hcg_refine_unionless",
    "hcg_shard_group_search_routed", "hcg_shard_group_local_shards",
]


class HcgScheme(C.Structure):
    _fields_ = [
        ("d_full", C.c_uint32),
        ("curves", C.c_uint32),
        ("bits_per_dim", C.c_uint32),
        ("curve_kind", C.c_uint32),
        ("assign_off", C.POINTER(C.c_uint32)),
        ("assign", C.POINTER(C.c_uint32)),
        ("cell_lut", C.c_uint32 * 256),
        ("dist_scale", C.c_double),
        ("dtype", C.c_uint32),
        ("view_offset", C.c_float),
    ]


class HcgNcclId(C.Structure):
    _fields_ = [("internal", C.c_uint8 * 128)]


class HcgServerPolicy(C.Structure):
    _fields_ = [("max_batch", C.c_uint32), ("min_batch", C.c_uint32), ("max_wait_s", C.c_double),
                ("slots", C.c_uint32)]


class HcgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[hcg {code}] {msg}")
        self.code = code


class HcgInvalidArgument(HcgError, ValueError):
    """Mirrors the reference's std::invalid_argument (curve.cpp:35-59, vecio.cpp:15,78,88,116)."""


class HcgIOError(HcgError):
    """Mirrors the reference's std::runtime_error for I/O (vecio.cpp:20-84)."""


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension must be built "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, u8, u32, u64 = C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64
    P = C.POINTER
    L.hcg_last_error.restype = C.c_char_p
    L.hcg_version.restype = C.c_char_p
    L.hcg_make_lut.argtypes = [C.c_float, C.c_float, u32, P(u32)]
    L.hcg_default_assignment.argtypes = [u32, u32, P(u32), P(u32)]
    L.hcg_build.argtypes = [P(HcgScheme), vp, u64, u64, u64, C.c_int, vp, P(vp)]
    L.hcg_free.argtypes = [vp]
    L.hcg_size.restype = u64
    L.hcg_size.argtypes = [vp]
    L.hcg_curves.restype = u32
    L.hcg_curves.argtypes = [vp]
    L.hcg_key_words.restype = u32
    L.hcg_key_words.argtypes = [vp, u32]
    L.hcg_device_bytes.restype = u64
    L.hcg_device_bytes.argtypes = [vp]
    L.hcg_launch_count.restype = u64
    L.hcg_launch_count.argtypes = []
    L.hcg_index_dtype.restype = u32
    L.hcg_index_dtype.argtypes = [vp]
    L.hcg_search.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, vp]
    L.hcg_search_timed.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, P(C.c_float), vp]
    L.hcg_search_packed.argtypes = [vp, vp, u32, u32, u32, vp, vp]
    L.hcg_merge_packed.argtypes = [vp, u32, u32, u32, vp, vp, vp, C.c_int, vp]
    L.hcg_keys.argtypes = [vp, vp, u64, u32, vp, vp]
    L.hcg_sorted.argtypes = [vp, u32, vp, vp, vp]
    L.hcg_sorted_range.argtypes = [vp, u32, u64, u64, vp, vp]
    L.hcg_describe.argtypes = [vp, P(HcgScheme), vp, vp, P(u32)]
    L.hcg_windows.argtypes = [vp, vp, u32, u32, vp, vp, vp, vp]
    L.hcg_candidates.argtypes = [vp, vp, u32, u32, vp, u32, vp, vp]
    L.hcg_brute_force.argtypes = [vp, vp, u32, u32, vp, vp, vp, vp]
    L.hcg_search_f32.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, vp]
    L.hcg_brute_force_f32.argtypes = [vp, vp, u32, u32, vp, vp, vp, vp]
    L.hcg_binomial_tail.restype = C.c_double
    L.hcg_binomial_tail.argtypes = [u32, C.c_double, u32]
    L.hcg_miss_bound.restype = C.c_double
    L.hcg_miss_bound.argtypes = [u32, u32, u32]
    L.hcg_plan_depth.restype = u32
    L.hcg_plan_depth.argtypes = [u32, u32, C.c_double]
    L.hcg_gen_rows.argtypes = [u64, u64, u64, vp, C.c_int, vp]
    L.hcg_gen_queries.argtypes = [u64, u64, u64, vp, C.c_int, vp]
    L.hcg_insert.argtypes = [vp, vp, u64, vp]
    L.hcg_save.argtypes = [vp, C.c_char_p]
    L.hcg_load.argtypes = [C.c_char_p, C.c_int, vp, P(vp)]
    L.hcg_read_vectors.argtypes = [C.c_char_p, u32, C.c_float, C.c_float, P(P(C.c_uint8)), P(u64), P(u32)]
    L.hcg_write_vectors.argtypes = [C.c_char_p, u32, C.c_float, C.c_float, vp, u64, u32]
    L.hcg_free_buffer.argtypes = [vp]
    L.hcg_free_buffer.restype = None
    L.hcg_nccl_unique_id.argtypes = [P(HcgNcclId)]
    L.hcg_shard_group_build.argtypes = [P(HcgScheme), vp, u64, u32, P(C.c_int), P(vp)]
    L.hcg_shard_group_adopt.argtypes = [u32, P(vp), P(vp)]
    L.hcg_shard_group_join.argtypes = [P(HcgNcclId), u32, u32, vp, P(vp)]
    L.hcg_shard_group_free.argtypes = [vp]
    L.hcg_shard_group_shards.restype = u32
    L.hcg_shard_group_shards.argtypes = [vp]
    L.hcg_shard_group_search.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, vp]
    L.hcg_shard_group_search_routed.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, vp, P(u32), P(u32)]
    L.hcg_index_device.restype = C.c_int
    L.hcg_index_device.argtypes = [vp]
    L.hcg_index_ids.argtypes = [vp, P(u64), P(u64)]
    L.hcg_refine_unionless.restype = u32
    L.hcg_refine_unionless.argtypes = [vp, u32, u32, u32]
    L.hcg_shard_group_device.restype = C.c_int
    L.hcg_shard_group_device.argtypes = [vp]
    L.hcg_shard_group_local_shards.restype = u32
    L.hcg_shard_group_local_shards.argtypes = [vp]
    L.hcg_shard_group_dims.restype = u32
    L.hcg_shard_group_dims.argtypes = [vp]
    L.hcg_server_create.argtypes = [vp, vp, u32, u32, P(HcgServerPolicy), P(vp)]
    L.hcg_server_free.argtypes = [vp]
    L.hcg_server_replay.argtypes = [vp, vp, u32, vp, vp, vp, vp, vp, vp, P(u32)]
    L.hcg_server_start.argtypes = [vp, u64]
    L.hcg_server_submit.argtypes = [vp, vp, u32, P(u64)]
    L.hcg_server_wait.argtypes = [vp, u64, vp, vp, vp, vp]
    for name in ("hcg_make_lut", "hcg_default_assignment", "hcg_build", "hcg_free", "hcg_search",
                 "hcg_search_timed", "hcg_search_packed", "hcg_merge_packed", "hcg_keys", "hcg_sorted", "hcg_windows",
                 "hcg_candidates", "hcg_brute_force", "hcg_search_f32", "hcg_brute_force_f32", "hcg_sorted_range",
                 "hcg_describe", "hcg_gen_rows", "hcg_gen_queries", "hcg_insert",
                 "hcg_save", "hcg_load", "hcg_read_vectors", "hcg_write_vectors", "hcg_nccl_unique_id",
                 "hcg_shard_group_build", "hcg_shard_group_adopt", "hcg_shard_group_join", "hcg_shard_group_free",
                 "hcg_shard_group_search", "hcg_shard_group_search_routed", "hcg_index_ids", "hcg_server_create", "hcg_server_free",
                 "hcg_server_replay", "hcg_server_start", "hcg_server_submit", "hcg_server_wait"):
        getattr(L, name).restype = C.c_int
    del u8
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == HCG_OK:
        return
    msg = lib().hcg_last_error().decode(errors="replace")
    if rc in (HCG_EINVAL, HCG_ECAPACITY, HCG_ENONFINITE):
        raise HcgInvalidArgument(rc, msg)
    if rc == HCG_EIO:
        raise HcgIOError(rc, msg)
    raise HcgError(rc, msg)
