"""The C ABI boundary without a GPU: the in-tree libhcg.so loads, exports every
entry point include/hcg.h declares, and its host-side pieces (LUT, scheme,
argument validation, planner) behave; compute calls are left to -m gpu."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1209_0410_b200 as H
from paper_1209_0410_b200 import _lib
from oracle import pyoracle as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hcg.h")).read()
    return sorted(set(re.findall(r"\b(hcg_[a-z_0-9]+)\s*\(", text)))


def test_library_is_in_tree_and_loads():
    assert os.path.dirname(_lib.LIB_PATH) == os.path.join(ROOT, "paper_1209_0410_b200")
    assert H.lib().hcg_version().decode().startswith("hcg")


def test_every_declared_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = C.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_lib_is_sm100a_only():
    """The fatbin carries sm_100a SASS and nothing else."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


@pytest.mark.parametrize("view", [H.RAW, H.LIFTED])
@pytest.mark.parametrize("m", [1, 8, 12, 16, 17, 24, 32])
def test_make_lut_matches_reference_quantizer(view, m):
    lut = H.make_lut(view, m)
    f = view.floats(np.arange(256, dtype=np.uint8))
    want = [P.quantize(float(x), m) for x in f]
    assert list(lut) == want


def test_make_lut_rejects_bad_m_and_nonfinite():
    lut = (C.c_uint32 * 256)()
    assert H.lib().hcg_make_lut(C.c_float(0), C.c_float(1), 0, lut) == _lib.HCG_EINVAL
    assert H.lib().hcg_make_lut(C.c_float(0), C.c_float(1), 33, lut) == _lib.HCG_EINVAL
    assert H.lib().hcg_make_lut(C.c_float(0), C.c_float(float("inf")), 8, lut) == _lib.HCG_ENONFINITE


def test_default_scheme_spec_examples():
    """SPEC.md:206-207."""
    assert H.default_scheme(4, 2).assignment == [[0, 2], [1, 3]]
    s = H.default_scheme(128, 8)
    assert [s.dims_of(c) for c in range(8)] == [16] * 8
    assert s.assignment[0][:3] == [0, 8, 16]
    with pytest.raises(ValueError):
        H.default_scheme(4, 5)        # curves > d_full
    with pytest.raises(ValueError):
        H.default_scheme(128, 8, seed=3)  # seeded permutation unpinned


def _scheme(d_full=128, curves=8, m=8, kind=1, assign=None):
    s = _lib.HcgScheme()
    sch = H.default_scheme(d_full, curves, m, kind)
    flat = assign if assign is not None else [a for row in sch.assignment for a in row]
    off = [0]
    for row in sch.assignment:
        off.append(off[-1] + len(row))
    s._off = (C.c_uint32 * len(off))(*off)
    s._asg = (C.c_uint32 * len(flat))(*flat)
    s.d_full, s.curves, s.bits_per_dim, s.curve_kind = d_full, curves, m, kind
    s.assign_off, s.assign = s._off, s._asg
    lut = H.make_lut(H.RAW, min(m, 32) if 1 <= m <= 32 else 8)
    for b in range(256):
        s.cell_lut[b] = int(lut[b])
    s.dist_scale = 1.0
    return s


def _build_rc(s, n=4):
    rows = np.zeros((n, s.d_full * 4), np.uint8)  # room for f32 rows too
    h = C.c_void_p()
    return H.lib().hcg_build(C.byref(s), rows.ctypes.data, n, 0, 1, 0, None, C.byref(h))


def test_build_validates_before_touching_the_device():
    assert _build_rc(_scheme(m=0)) == _lib.HCG_EINVAL
    assert _build_rc(_scheme(kind=7)) == _lib.HCG_EINVAL
    assert _build_rc(_scheme(curves=1, m=16)) == _lib.HCG_ECAPACITY  # 2048-bit key
    bad = _scheme()
    bad._asg[0] = 500
    assert _build_rc(bad) == _lib.HCG_EINVAL
    uncovered = _scheme(d_full=4, curves=2, assign=[0, 0, 1, 3])
    assert _build_rc(uncovered) == _lib.HCG_EINVAL
    msg = H.lib().hcg_last_error().decode()
    assert "covered" in msg


def test_f32_scheme_validation():
    s = _scheme()
    s.dtype = 2
    assert _build_rc(s) == _lib.HCG_EINVAL  # unknown dtype
    wide = _scheme(d_full=129, curves=3)
    wide.dtype = _lib.HCG_F32  # 129 floats = 516 bytes > HCG_MAX_ROW_BYTES
    assert _build_rc(wide) == _lib.HCG_ECAPACITY
    assert "128" in H.lib().hcg_last_error().decode()
    m32 = _scheme(curves=8, m=32)
    m32.dtype = _lib.HCG_F32
    for b in range(256):
        m32.cell_lut[b] = 0xFFFFFFFF  # the table is unused for float rows
    assert _build_rc(m32) in (_lib.HCG_OK, _lib.HCG_ENODEV)


def test_no_gpu_is_an_error_not_a_fallback():
    from hcg_testutil import gpu_available
    if gpu_available():
        pytest.skip("a GPU is present")
    assert _build_rc(_scheme()) == _lib.HCG_ENODEV
    with pytest.raises(_lib.HcgError):
        H.MulticurvesIndex(np.zeros((10, 128), np.uint8), H.default_scheme(128, 8))


def test_planner_host_functions():
    assert H.plan_depth(175, 2, 0.02) == 113
    assert H.shard_probe_depth(350, 8) == 80
    assert H.miss_bound(10, 1, 5) == 1.0
    with pytest.raises(ValueError):
        H.binomial_tail(10, 1.5, 3)


@pytest.mark.parametrize("offset,scale,ok", [
    (0.0, 1.0, True),            # raw bytes
    (1.0, 1.0 / 256, True),      # lifted
    (-64.0, 0.5, True),          # any exact power-of-two view
    (0.0, 0.1, False),           # not a power of two: sqrt(S) * scale would round differently
    (0.0, 3.0, False),
    (1e8, 1.0, False),           # 1e8 + b is not exact in float32
])
def test_u8_view_must_be_exact(offset, scale, ok):
    """A u8 index reports sqrt(S) * scale for the integer S; that is the
    reference's rooted double only for views whose floats are exact and whose
    scale is a power of two, so other views are rejected up front (before any
    device work, so this runs without a GPU)."""
    s = _scheme()
    s.dist_scale = scale
    s.view_offset = offset
    rc = _build_rc(s)
    if ok:
        assert rc in (_lib.HCG_OK, _lib.HCG_ENODEV)
    else:
        assert rc == _lib.HCG_EINVAL
        assert b"u8 view" in H.lib().hcg_last_error()


def test_shard_group_validation_without_a_device():
    """hcg_shard_group_*: argument checks come before NCCL or the device."""
    L = H.lib()
    h = C.c_void_p()
    assert L.hcg_shard_group_adopt(0, None, C.byref(h)) == _lib.HCG_EINVAL
    s = _scheme()
    assert L.hcg_shard_group_build(C.byref(s), None, 10, 2, None, C.byref(h)) == _lib.HCG_EINVAL
    devs = (C.c_int * 2)(0, 1)
    s32 = _scheme()
    s32.dtype = _lib.HCG_F32
    assert L.hcg_shard_group_build(C.byref(s32), None, 0, 2, devs, C.byref(h)) == _lib.HCG_EINVAL
    nid = _lib.HcgNcclId()
    assert L.hcg_shard_group_join(C.byref(nid), 2, 2, None, C.byref(h)) == _lib.HCG_EINVAL
    q = np.zeros((1, 128), np.uint8)
    assert L.hcg_shard_group_search(None, q.ctypes.data, 1, 10, 10, None, None, None, None) == _lib.HCG_EINVAL
    assert L.hcg_shard_group_shards(None) == 0
    assert L.hcg_index_device(None) == -1
