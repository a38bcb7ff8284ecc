"""bvecs / fvecs records (vecio.cpp:18-85): the library's reader
and writer against the reference's own read_vectors (oracle/_ref) -- same
payload, same rejection of malformed files (std::runtime_error <-> HcgIOError)."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

import paper_1209_0410_b200 as H
from oracle import pyoracle as P


def ref_read(path, bvecs):
    lib = P.ref()
    lib.ref_read_vectors.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint32)]
    out = np.zeros(1 << 16, np.float32)
    n, d = C.c_uint64(), C.c_uint32()
    rc = lib.ref_read_vectors(os.fsencode(path), int(bvecs), out.ctypes.data, out.size, C.byref(n), C.byref(d))
    return rc, out[: n.value * d.value].reshape(n.value, d.value) if rc == 0 else None


@pytest.mark.parametrize("fmt,view", [("bvecs", H.RAW), ("fvecs", H.RAW), ("fvecs", H.LIFTED)])
def test_round_trip_and_reference_reader(tmp_path, fmt, view):
    rows = np.random.default_rng(1).integers(0, 256, (300, 128), dtype=np.uint8)
    path = str(tmp_path / f"x.{fmt}")
    H.write_vectors(path, rows, fmt, view)
    back = H.read_vectors(path, fmt, view)
    np.testing.assert_array_equal(back, rows)
    if P.ref_available():
        rc, f = ref_read(path, fmt == "bvecs")
        assert rc == 0
        want = view.floats(rows) if fmt == "fvecs" else rows.astype(np.float32)
        np.testing.assert_array_equal(f, want)


def test_empty_file_is_empty_dataset(tmp_path):
    p = tmp_path / "e.bvecs"
    p.write_bytes(b"")
    assert H.read_vectors(str(p)).shape[0] == 0


@pytest.mark.parametrize("payload,why", [
    (struct.pack("<I", 4) + b"\x01\x02", "truncated bvecs payload"),
    (struct.pack("<I", 4) + b"\x01\x02\x03\x04" + b"\x01\x00", "truncated record header"),
    (struct.pack("<I", 0), "zero-dimension record"),
    (struct.pack("<I", 2) + b"ab" + struct.pack("<I", 3) + b"abc", "inconsistent dimension header"),
])
def test_malformed_files_rejected_like_the_reference(tmp_path, payload, why):
    p = tmp_path / "bad.bvecs"
    p.write_bytes(payload)
    with pytest.raises(H.HcgIOError, match=why):
        H.read_vectors(str(p))
    if P.ref_available():
        rc, _ = ref_read(str(p), True)
        assert rc != 0 and why in P.ref_error()


def test_nonfinite_fvecs_rejected(tmp_path):
    p = tmp_path / "nan.fvecs"
    p.write_bytes(struct.pack("<I", 2) + struct.pack("<2f", 1.0, float("nan")))
    with pytest.raises(H.HcgIOError, match="non-finite"):
        H.read_vectors(str(p), "fvecs")


def test_missing_file(tmp_path):
    with pytest.raises(H.HcgIOError, match="cannot open"):
        H.read_vectors(str(tmp_path / "nope.bvecs"))


def test_float_fvecs_round_trip_and_reference_reader(tmp_path):
    """fvecs with arbitrary float components (rows of an HCG_F32 index): the
    payload is kept bit-for-bit and equals what the reference's reader loads."""
    rng = np.random.default_rng(2)
    rows = (rng.standard_normal((257, 96)) * 1e3).astype(np.float32)
    rows[0, :4] = [0.0, -0.0, 1e-40, -3.4e38]  # zeros, a denormal, a large value
    path = str(tmp_path / "f.fvecs")
    H.write_vectors(path, rows, "fvecs")
    back = H.read_vectors(path, "fvecs", dtype="f32")
    assert back.dtype == np.float32 and back.tobytes() == rows.tobytes()
    if P.ref_available():
        rc, f = ref_read(path, False)
        assert rc == 0 and f.tobytes() == rows.tobytes()
    p = tmp_path / "nan.fvecs"
    p.write_bytes(struct.pack("<I", 2) + struct.pack("<2f", 1.0, float("inf")))
    with pytest.raises(H.HcgIOError, match="non-finite"):
        H.read_vectors(str(p), "fvecs", dtype="f32")
    with pytest.raises(H.HcgInvalidArgument):
        H.read_vectors(path, "bvecs", dtype="f32")


def test_search_csv_round_trip(tmp_path):
    """cmd_search's `query_id,rank,neighbor_id,distance` rows:
    one row per neighbour in list order; doubles round-trip exactly."""
    ids = np.array([[7, 3, 2**64 - 1], [1, 2, 5]], np.uint64)
    d = np.array([[0.0, np.sqrt(2.0), np.inf], [1.0 / 3, 2.5, 1e-300]])
    lens = np.array([2, 3], np.uint32)
    p = str(tmp_path / "r.csv")
    assert H.write_search_csv(p, ids, d, lens, query_ids=[10, 11]) == 5
    rows = H.read_search_csv(p)
    assert [r[:3] for r in rows] == [(10, 0, 7), (10, 1, 3), (11, 0, 1), (11, 1, 2), (11, 2, 5)]
    assert [r[3] for r in rows] == [0.0, np.sqrt(2.0), 1.0 / 3, 2.5, 1e-300]
    (tmp_path / "bad.csv").write_text("a,b\n")
    with pytest.raises(H.HcgInvalidArgument):
        H.read_search_csv(str(tmp_path / "bad.csv"))
